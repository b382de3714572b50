"""The user-facing end of the synthesizer: reports (the JSON document -- schema version 1,
byte-stable for identical inputs -- a text rendering, the per-op constraint trace behind
``--explain``) and the ``tilesynth`` command line that produces them.

Contract: /root/reference/pkg/src/tilesynth/report.py:1-289 -- the JSON keys, nesting, value
formats (layouts as ``shape:stride`` text, swizzles as ``SW(b,b,s)``, conflicts keyed by the op
index as a string) and ``json.dumps(indent=2, sort_keys=True)`` + newline, so reports compare
byte for byte. The text and explain renderings are this package's own. The command line keeps the
reference CLI's flags, defaults and exit codes (/root/reference/pkg/src/tilesynth/cli.py): 0 success,
1 diagnostics / synthesis failure / malformed input, 2 usage error (bad flags, unreadable files);
no environment variables are consulted.

    version, arch, threads, program{ops, tensors{name: {scope, dtype, shape}}},
    candidates{count, costs}, best{index, total_cycles, tensors{name: {tv, tile}},
    copies[{op, instruction, vector_bytes, conflicts?, identity_conflicts?}],
    buffers{name: {layout, swizzle, conflicts, identity_conflicts}},
    redistributions[{op, tensor, from, to}],
    cost[{label, instruction, invocations, issue, stall, start, completes}]}, all?, diagnostics
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

from .algebra import compose, dim_restrict, group_modes, inverse
from .errors import CatalogFormatError, ParseError, UnknownOp
from .explore import synthesize_program
from .isa_table import builtin_catalog_path, load_catalog
from .layout_flow import SynthesisConfig, slot_for
from .smem_plan import build_constraint
from .tileprog import parse_program
from .algebra import restrict_tv

SCHEMA_VERSION = 1


_COST_FIELDS = ("label", "instruction", "invocations", "issue", "stall", "start", "completes")


def _gemm_lines(graph, cand, op):
    inst = cand.choices[op.index]
    (mi, ni, ki), (m, k), n = inst.mnk, graph.tensor(op.operands[0]).shape, graph.tensor(op.operands[1]).shape[0]
    pa, pb, pc = inst.mma_layouts()
    ca, cb, cc = (_through_instruction(cand.layouts[t], p) for t, p in zip(op.operands, (pa, pb, pc)))
    lines = [f"  instruction {inst.name} tile {mi}x{ni}x{ki}"]
    # (equation, left map, its in/out dims and extents, right map, its in/out dims and extents)
    for label, left, lspec, right, rspec in (
            ("rows", cc, (0, 0, (mi, ni), (m, n)), ca, (0, 0, (mi, ki), (m, k))),
            ("cols", cc, (1, 1, (mi, ni), (m, n)), cb, (0, 0, (ni, ki), (n, k))),
            ("reduction", ca, (1, 1, (mi, ki), (m, k)), cb, (1, 1, (ni, ki), (n, k)))):
        lhs, rhs = dim_restrict(left, *lspec), dim_restrict(right, *rspec)
        lines.append(f"  {label}: {lhs} == {rhs}  [{'ok' if lhs.equivalent(rhs) else 'MISMATCH'}]")
    return lines


def _copy_lines(graph, cand, op):
    src, dst = op.operands[0], op.results[0]
    f, g = (cand.layouts[slot_for(graph, op, t)] for t in (src, dst))
    lines = [f"  source {src}: {f.layout}", f"  dest   {dst}: {g.layout}"]
    inst = cand.choices.get(op.index)
    if inst is None:
        return lines + ["  register move: source and destination layouts equal"]
    p, q = inst.copy_layouts(graph.tensor(src).dtype)
    lines += [f"  instruction {inst.name}: p={p.layout}, q={q.layout}",
              "  rule: f composed with inverse(p) == g composed with inverse(q)"]
    for name, tv in ((src, f), (dst, g)):
        decl = graph.tensor(name)
        if decl.scope != "Shared":
            continue
        lines.append(f"  {name} layout constraint: {build_constraint(tv, inst.vector_elems(decl.dtype), decl.shape)}")
        if name in cand.smem:
            smem = cand.smem[name]
            lines += [f"  unified constraint: {smem.constraint}", f"  materialized: {smem.layout} (+) {smem.swizzle}"]
    return lines


def _elementwise_lines(graph, cand, op):
    return [f"  {t}: {cand.layouts[t].layout}" for t in op.operands + op.results] + [
        "  rule: all operands share one thread-value layout"]


def _reduce_lines(graph, cand, op):
    f, g = (cand.layouts[t].layout for t in (op.operands[0], op.results[0]))
    return [f"  input  {op.operands[0]}: {f}", f"  output {op.results[0]}: {g}",
            f"  rule: collapse dimension {op.reduce_dim} of the input map"]


_EXPLAIN = {"gemm": _gemm_lines, "copy": _copy_lines, "reduce": _reduce_lines, "cast": _elementwise_lines,
            "elementwise": _elementwise_lines}


# ---------------------------------------------------------------------------------------- command line
_FLAGS = (
    (("--program",), dict(required=True, help="program file")),
    (("--catalog",), dict(default=None, help="instruction catalog file (default: bundled sm80 catalog)")),
    (("--threads",), dict(type=int, default=128, help="threads per tile (default 128)")),
    (("--max-candidates",), dict(type=int, default=64, help="search-tree leaf cap (default 64)")),
    (("--report",), dict(default=None, help="write the report to this path")),
    (("--format",), dict(choices=("json", "text"), default="text")),
    (("--explain",), dict(type=int, default=None, metavar="OP",
                          help="print the constraint trace for one operation and exit")),
    (("--all-candidates",), dict(action="store_true", help="include every surviving search leaf in the report")),
)


class _Exit(Exception):
    def __init__(self, code, message=""):
        super().__init__(message)
        self.code, self.message = code, message


def main(argv=None):
    args = _parser().parse_args(argv)
    try:
        return _run(args)
    except _Exit as stop:
        if stop.message:
            print(stop.message, file=sys.stderr)
        return stop.code


if __name__ == "__main__":
    sys.exit(main())


def build_report(result, all_candidates=False):
    """The report dict. A catalog with TMA entries (sm100) adds ``best.buffers[name].tma``: whether
    the bulk tensor engine can serve the buffer (smem_plan.check_tma on its unified constraint);
    catalogs without them (sm80) produce the reference's schema unchanged."""
    g = result.graph
    out = {
        "version": SCHEMA_VERSION,
        "arch": result.catalog.arch,
        "threads": result.config.threads,
        "program": {"ops": len(g.ops),
                    "tensors": {n: {"scope": d.scope, "dtype": str(d.dtype), "shape": list(d.shape)}
                                for n, d in sorted(g.tensors.items())}},
        "diagnostics": list(result.diagnostics),
        "candidates": {"count": len(result.candidates), "costs": [c.cost.total_cycles for c in result.candidates]},
    }
    if result.best is not None:
        out["best"] = _candidate_section(result, result.best)
        from .repack import tma_plan
        for name, entry in tma_plan(result).items():
            out["best"]["buffers"][name]["tma"] = entry
    if all_candidates:
        out["all"] = [_candidate_section(result, c) for c in result.candidates]
    return out


def render_json(report):
    return json.dumps(report, indent=2, sort_keys=True) + "\n"


def render_text(report):
    """Human-readable summary of a report dict: a header, then one table per section of the best
    candidate (tensor layouts, copies, shared buffers, redistributions, cost steps)."""
    prog, cands, best = report["program"], report["candidates"], report.get("best")
    out = [f"tilesynth -- {report['arch']}, {report['threads']} threads, {prog['ops']} ops over "
           f"{len(prog['tensors'])} tensors; {cands['count']} candidates {cands['costs']}"]
    out += [f"diagnostic: {d}" for d in report["diagnostics"]]
    if best:
        out.append(f"best candidate #{best['index']}: {best['total_cycles']} cycles")
        sections = (
            ("register / tensor layouts", ("tensor", "thread-value layout", "tile"),
             [(f"{n}:", t["tv"], "x".join(map(str, t["tile"]))) for n, t in best["tensors"].items()]),
            ("copies", ("op", "instruction", "bytes", "conflicts (identity)"),
             [(c["op"], c["instruction"], c["vector_bytes"],
               f"{c['conflicts']} ({c['identity_conflicts']})" if "conflicts" in c else "-") for c in best["copies"]]),
            ("shared buffers", ("buffer", "layout (+) swizzle", "tma"),
             [(f"{n}:", f"{b['layout']} (+) {b['swizzle']}",
               ("yes" if b["tma"]["feasible"] else "no") if "tma" in b else "-") for n, b in best["buffers"].items()]),
            ("redistributions", ("op", "tensor", "from -> to"),
             [(r["op"], r["tensor"], f"{r['from']} -> {r['to']}") for r in best["redistributions"]]),
            ("cost", ("step", "instruction", "n", "issue", "stall", "start", "completes"),
             [(c["label"], c["instruction"], c["invocations"], c["issue"], c["stall"], c["start"], c["completes"])
              for c in best["cost"]]),
        )
        for title, header, rows in sections:
            out += _table(title, header, rows)
    return "\n".join(out) + "\n"


def explain_op(result, op_index):
    """The constraints touching one op, evaluated on the best candidate."""
    ops = result.graph.ops
    if op_index < 0 or op_index >= len(ops):
        raise UnknownOp(f"op index {op_index} out of range (0..{len(ops) - 1})")
    if result.best is None:
        return "no valid candidate to explain"
    op = ops[op_index]
    head = f"op {op_index}: {op.kind} {' '.join(op.operands)} -> {' '.join(op.results)}"
    body = _EXPLAIN.get(op.kind, lambda g, c, o: ["  redistribution step (no layout constraint)"])(
        result.graph, result.best, op)
    return "\n".join([head] + body) + "\n"


def _run(args):
    graph, cat = _inputs(args)
    result = synthesize_program(graph, cat, SynthesisConfig(threads=args.threads, max_candidates=args.max_candidates))
    diag_lines = "\n".join(f"diagnostic: {d}" for d in result.diagnostics)
    if args.explain is not None:
        if result.diagnostics:
            raise _Exit(1, diag_lines)
        try:
            sys.stdout.write(explain_op(result, args.explain))
        except UnknownOp as e:
            raise _Exit(1, f"error: {e}") from None
        return 0
    report = build_report(result, all_candidates=args.all_candidates)
    text = (render_json if args.format == "json" else render_text)(report)
    if args.report:
        Path(args.report).write_text(text)
    else:
        sys.stdout.write(text)
    if not result.ok:
        raise _Exit(1, diag_lines)
    return 0


def _inputs(args):
    program = Path(args.program)
    catalog = Path(args.catalog) if args.catalog else builtin_catalog_path()
    for path, what in ((program, "program"), (catalog, "catalog")):
        if not path.is_file():
            raise _Exit(2, f"error: {what} file not found: {path}")
    if args.threads < 32 or args.threads % 32:
        raise _Exit(2, "error: --threads must be a positive multiple of 32")
    try:
        cat = load_catalog(catalog)
    except CatalogFormatError as e:
        raise _Exit(1, f"error: {e}") from None
    try:
        graph = parse_program(program.read_text())
    except ParseError as e:
        raise _Exit(1, f"error: {program}: {e}") from None
    return graph, cat


def _parser():
    p = argparse.ArgumentParser(prog="tilesynth", description="Synthesize thread-value and shared-memory layouts "
                                "for a tile-level GPU program and rank instruction choices by modeled latency.")
    for names, kw in _FLAGS:
        p.add_argument(*names, **kw)
    return p


# ------------------------------------------------------------------------------------------ explain
def _through_instruction(tv, inst_tv):
    """Known layout restricted to one instruction tile, composed with the instruction's inverse
    regrouped by its tile extents: instruction-tile coordinate -> tensor position."""
    core = restrict_tv(tv, inst_tv.threads, inst_tv.values)[0]
    return compose(core.layout, group_modes(inverse(inst_tv.layout), inst_tv.tile))


def _table(title, header, rows):
    """A titled, column-aligned block (no block for no rows)."""
    if not rows:
        return []
    cells = [header] + [[str(c) for c in r] for r in rows]
    widths = [max(len(r[i]) for r in cells) for i in range(len(header))]
    fmt = lambda r: "  " + "  ".join(c.ljust(w) for c, w in zip(r, widths)).rstrip()  # noqa: E731
    return [title] + [fmt(r) for r in cells]


def _candidate_section(result, cand):
    g = result.graph
    buffers = {name: _buffer_entry(s) for name, s in sorted(cand.smem.items())}
    buffers.update((name, _buffer_entry(s)) for name, s in sorted(cand.staging.items()))
    return {
        "index": cand.index,
        "total_cycles": cand.cost.total_cycles,
        "tensors": {name: {"tv": str(cand.layouts[name].layout), "tile": list(cand.layouts[name].tile)}
                    for name in sorted(g.tensors) if name in cand.layouts},
        "copies": [_copy_entry(g, cand, op) for op in g.ops
                   if op.kind == "copy" and op.index in cand.choices and cand.choices[op.index].category == "copy"],
        "buffers": buffers,
        "redistributions": [{"op": p.op_index, "tensor": p.tensor, "from": str(p.from_layout.layout),
                             "to": str(p.to_layout.layout)} for p in cand.patches],
        "cost": [{k: getattr(row, k) for k in _COST_FIELDS} for row in cand.cost.breakdown],
    }


def _copy_entry(graph, cand, op):
    inst = cand.choices[op.index]
    entry = {"op": op.index, "instruction": inst.name, "vector_bytes": inst.vector_bytes}
    for name in (op.operands[0], op.results[0]):
        if name in cand.smem and graph.tensor(name).scope == "Shared":
            entry["conflicts"] = cand.smem[name].copy_conflicts.get(op.index)
            entry["identity_conflicts"] = cand.smem[name].identity_conflicts.get(op.index)
    return entry


def _buffer_entry(smem):
    return {
        "layout": str(smem.layout),
        "swizzle": str(smem.swizzle),
        "conflicts": {str(k): v for k, v in sorted(smem.copy_conflicts.items())},
        "identity_conflicts": {str(k): v for k, v in sorted(smem.identity_conflicts.items())},
    }

"""Differential fuzzing of the synthesizer's building blocks against the REFERENCE implementation
(imported read-only from /root/reference/pkg/src when present -- build container only; the committed
goldens in test_tilesynth_parity.py carry parity everywhere else).

Each case draws random operands (bijective layouts, strided sub-samplings, nested trees, TV layouts,
constraints, access patterns) and requires the same result string -- or the same error class -- from
both implementations."""
import importlib
import random
import sys

import pytest

pytestmark = pytest.mark.reference


@pytest.fixture(scope="module")
def ref():
    sys.path.insert(0, "/root/reference/pkg/src")
    try:
        mods = {m: importlib.import_module(f"tilesynth.{m}") for m in ("layout", "tv", "swizzle", "smem", "inttuple")}
    finally:
        sys.path.remove("/root/reference/pkg/src")
    return mods


from paper_2504_16214_b200.tilesynth import smem_plan as B  # noqa: E402
from paper_2504_16214_b200.tilesynth import algebra as LA  # noqa: E402
from paper_2504_16214_b200.tilesynth import ituple as N  # noqa: E402
from paper_2504_16214_b200.tilesynth import smem_plan as SM  # noqa: E402
from paper_2504_16214_b200.tilesynth import algebra as TV  # noqa: E402


def _outcome(fn, *args):
    try:
        r = fn(*args)
    except Exception as e:  # noqa: BLE001
        return ("error", type(e).__name__)
    if isinstance(r, tuple):
        return tuple(str(x) for x in r)
    return str(r)


def _rand_tree(rng, leaves, depth=0):
    """Random nesting of a flat list of leaves."""
    if len(leaves) <= 1 or depth > 2 or rng.random() < 0.3:
        return tuple(leaves) if len(leaves) > 1 or rng.random() < 0.5 else leaves[0]
    cut = rng.randint(1, len(leaves) - 1)
    return (_rand_tree(rng, leaves[:cut], depth + 1), _rand_tree(rng, leaves[cut:], depth + 1))


def _regroup(rng, shapes, strides):
    """Same leaves, random (identical) nesting for shape and stride."""
    idx = list(range(len(shapes)))
    tree = _rand_tree(rng, idx)
    tree = tree if isinstance(tree, tuple) else (tree,)

    def sub(t, vals):
        return vals[t] if isinstance(t, int) else tuple(sub(c, vals) for c in t)
    return sub(tree, shapes), sub(tree, strides)


def _bijective(rng, max_size=256):
    shapes, total = [], 1
    for _ in range(rng.randint(1, 5)):
        s = rng.choice([1, 2, 2, 3, 4, 8])
        if total * s > max_size:
            break
        shapes.append(s)
        total *= s
    shapes = shapes or [2]
    order = list(range(len(shapes)))
    rng.shuffle(order)
    strides, w = [0] * len(shapes), 1
    for i in order:
        strides[i], w = w, w * shapes[i]
    return _regroup(rng, shapes, strides)


def _any_layout(rng):
    n = rng.randint(1, 4)
    shapes = [rng.choice([1, 2, 3, 4, 8]) for _ in range(n)]
    strides = [rng.choice([0, 1, 2, 3, 4, 8, 16, 32]) for _ in range(n)]
    return _regroup(rng, shapes, strides)


def test_layout_algebra_matches_reference(ref):
    L = ref["layout"]
    rng = random.Random(0xD1FF)
    for _ in range(4000):
        sa, da = _bijective(rng) if rng.random() < 0.7 else _any_layout(rng)
        sb, db = _any_layout(rng) if rng.random() < 0.5 else _bijective(rng, 64)
        ours_a, ours_b = LA.Layout(sa, da), LA.Layout(sb, db)
        ref_a, ref_b = L.Layout(sa, da), L.Layout(sb, db)
        assert _outcome(LA.coalesce, ours_a) == _outcome(L.coalesce, ref_a)
        assert _outcome(LA.compose, ours_a, ours_b) == _outcome(L.compose, ref_a, ref_b), (sa, da, sb, db)
        assert _outcome(LA.inverse, ours_a) == _outcome(L.inverse, ref_a), (sa, da)
        m = ours_a.size() * rng.choice([1, 2, 3, 4])
        assert _outcome(LA.complement, ours_a, m) == _outcome(L.complement, ref_a, m), (sa, da, m)
        mode = rng.randrange(ours_a.rank)
        n = rng.randint(1, max(1, N.size(sa[mode] if isinstance(sa, tuple) else sa)))
        assert _outcome(LA.restrict_mode_split, ours_a, mode, n) == _outcome(L.restrict_mode_split, ref_a, mode, n)
        total = ours_a.size()
        divs = [d for d in range(1, total + 1) if total % d == 0]
        g = rng.choice(divs)
        sizes = (g, total // g) if rng.random() < 0.8 else (g, max(1, total // g // 2), 2)
        assert _outcome(LA.group_modes, ours_a, sizes) == _outcome(L.group_modes, ref_a, sizes), (sa, da, sizes)
        x = rng.randrange(total) if total else 0
        assert ours_a(x) == ref_a(x)


def test_tuple_parsing_matches_reference(ref):
    it = ref["inttuple"]
    rng = random.Random(7)
    alphabet = "(),0123 "
    samples = ["(2,)", "()", "(2,3))", "((2,4),(2,2))", "7", "(1)", "((1))", "(2,(3,4),5)", "", "(2 3)", "(,2)",
               "((2),)", "(2,3", "x", "(-1)"]
    samples += ["".join(rng.choice(alphabet) for _ in range(rng.randint(0, 10))) for _ in range(3000)]
    for s in samples:
        assert _outcome(N.parse_tuple, s) == _outcome(it.parse_tuple, s), repr(s)


def test_tv_and_bank_model_match_reference(ref):
    tv_ref, sw_ref = ref["tv"], ref["swizzle"]
    rng = random.Random(11)
    for _ in range(300):
        sa, da = _bijective(rng, 512)
        lay = LA.Layout(sa, da)
        size = lay.size()
        t = rng.choice([d for d in range(1, size + 1) if size % d == 0])
        try:
            grouped = LA.group_modes(lay, (t, size // t))
        except Exception:  # noqa: BLE001
            continue
        ours = TV.TvLayout(grouped, (size,))
        theirs = tv_ref.TvLayout(ref["layout"].Layout(grouped.shape, grouped.stride), (size,))
        assert str(TV.filter_replication(ours).layout) == str(tv_ref.filter_replication(theirs).layout)
        assert _outcome(TV.restrict_tv, ours, 1, 1)[0] == _outcome(tv_ref.restrict_tv, theirs, 1, 1)[0]
    for _ in range(2000):
        width = rng.choice([1, 2, 4, 8, 16])
        lanes = rng.choice([32, 32, 32, 8, 5])
        addrs = tuple(width * rng.randrange(0, 512) for _ in range(lanes))
        sw = rng.choice(B.candidate_swizzles())
        ref_sw = sw_ref.Swizzle(sw.bits, sw.base, sw.shift)
        got = _outcome(B.bank_conflicts, B.AccessPattern(addrs, width), sw)
        want = _outcome(sw_ref.bank_conflicts, sw_ref.AccessPattern(addrs, width), ref_sw)
        assert got == want, (addrs, width, sw)


def test_constraint_unify_materialize_match_reference(ref):
    S = ref["smem"]
    rng = random.Random(5)
    texts = []
    for _ in range(1500):
        dims = [rng.choice([8, 16, 32, 64]) for _ in range(rng.randint(1, 2))]
        parts, var = [], 0
        for d in dims:
            pieces, left = [], d
            while left > 1:
                p = rng.choice([q for q in (2, 4, 8) if left % q == 0] or [left])
                pieces.append(p)
                left //= p
            strides = []
            for _p in pieces:
                if rng.random() < 0.4:
                    strides.append(str(rng.choice([1, 2, 4, 8, 16, 32, 64])))
                else:
                    var += 1
                    strides.append(f"D{var}")
            parts.append((pieces, strides))
        shape = ",".join(f"({','.join(map(str, p))})" if len(p) > 1 else str(p[0]) for p, _ in parts)
        stride = ",".join(f"({','.join(s)})" if len(s) > 1 else s[0] for _, s in parts)
        texts.append(f"({shape}):({stride})")
    for a, b in zip(texts, texts[1:] + texts[:1]):
        ours_a, ours_b = SM.parse_constraint(a), SM.parse_constraint(b)
        ref_a, ref_b = S.parse_constraint(a), S.parse_constraint(b)
        assert _outcome(SM.materialize, ours_a) == _outcome(S.materialize, ref_a), a
        u1, u2 = _outcome(SM.unify, ours_a, ours_b), _outcome(S.unify, ref_a, ref_b)
        assert u1 == u2, (a, b)
        tma = lambda mod, c: (lambda r: (r.feasible, str(r.hint)))(mod.check_tma(c, 16))  # noqa: E731
        assert _outcome(tma, SM, ours_a) == _outcome(tma, S, ref_a), a


def _random_program(rng) -> tuple[str, int]:
    """A random tile program from a few families (copy chains, GEMM tiles, int4 weight tiles, reductions,
    rearranges), random extents / layouts / dtypes; returns (text, threads)."""
    threads = rng.choice([32, 64, 128, 128, 256])
    fam = rng.choice(["copy", "gemm", "int4", "reduce", "rearrange", "gemm"])
    if fam == "copy":
        m, n = rng.choice([16, 32, 64, 128]), rng.choice([16, 32, 64])
        dt = rng.choice(["float16", "float32", "int8", "bfloat16"])
        col = rng.random() < 0.3
        lay = f"({m},{n}):(1,{m})" if col else f"({m},{n}):({n},1)"
        mid = rng.choice(["register_tensor", "shared_tensor"])
        text = (f"gi = global_view a {dt} {lay}\ngo = global_view b {dt} ({m},{n}):({n},1)\n"
                f"t = {mid} {dt} ({m},{n})\nr = register_tensor {dt} ({m},{n})\n")
        text += "copy gi t\ncopy t r\ncopy r go\n" if mid == "shared_tensor" else "copy gi t\ncopy t go\n"
        return text, threads
    if fam in ("gemm", "int4"):
        M = rng.choice([16, 32, 64, 128])
        N = rng.choice([32, 64, 128])
        K = rng.choice([16, 32, 64])
        wd = "int4" if fam == "int4" else "float16"
        if fam == "int4":
            gw = rng.choice([f"({N},{K}):({K},1)", f"({N},{K}):(1,{N})",
                             f"((8,{N // 8}),(2,4,{K // 8})):((8*0+{K},{8 * K}),(1,{K // 4 if K >= 32 else 1},2))"])
            gw = gw if "*" not in gw else f"({N},{K}):({K},1)"
        else:
            gw = f"({N},{K}):({K},1)"
        loop = rng.choice([1, 2, 4])
        text = (f"ga = global_view bA float16 ({M},{K}):({K},1)\ngw = global_view bW {wd} {gw}\n"
                f"gc = global_view bC float16 ({M},{N}):({N},1)\nra = register_tensor float16 ({M},{K})\n"
                f"sw = shared_tensor {wd} ({N},{K})\nw4 = register_tensor {wd} ({N},{K})\n"
                f"acc = register_tensor float32 ({M},{N})\n")
        body = "copy ga ra\ncopy gw sw\ncopy sw w4\n"
        body += "w16 = cast w4 float16\ngemm acc ra w16\n" if wd == "int4" else "gemm acc ra w4\n"
        text += (f"loop {loop}\n" + body + "endloop\n") if loop > 1 else body
        text += "c16 = cast acc float16\ncopy c16 gc\n"
        if rng.random() < 0.3:
            text += f"annotate {4 if wd == 'int4' else 3} thread_arrangement ({threads // 32},1):(1,{threads // 32})\n"
        return text, threads
    if fam == "reduce":
        m, n = rng.choice([32, 64]), rng.choice([8, 16, 32])
        return (f"gi = global_view a float32 ({m},{n}):({n},1)\ngo = global_view b float32 ({m},1):(1,{m})\n"
                f"r = register_tensor float32 ({m},{n})\ncopy gi r\nr2 = reduce r 1\ncopy r2 go\n"), threads
    m = rng.choice([32, 64])
    return (f"gin = global_view bi float32 ({m},32):(32,1)\ngout = global_view bo float32 ({m},32):(32,1)\n"
            f"r1 = register_tensor float32 ({m},32)\ncopy gin r1\n"
            f"r2 = rearrange r1 (({threads}),({m * 32 // threads})):((1),({threads})),\ncopy r2 gout\n"
            .replace("),\n", ")\n")), threads


def test_whole_synthesis_matches_reference_on_random_programs(ref):
    """Random programs through both synthesizers in one process: identical JSON reports (or the same
    parse / synthesis failure)."""
    sys.path.insert(0, "/root/reference/pkg/src")
    try:
        r_cat = importlib.import_module("tilesynth.catalog")
        r_ir = importlib.import_module("tilesynth.ir")
        r_pipe = importlib.import_module("tilesynth.pipeline")
        r_rep = importlib.import_module("tilesynth.report")
        r_synth = importlib.import_module("tilesynth.synth")
    finally:
        sys.path.remove("/root/reference/pkg/src")
    from paper_2504_16214_b200.tilesynth import isa_table as C
    from paper_2504_16214_b200.tilesynth import frontend as R
    from paper_2504_16214_b200.tilesynth import tileprog as IR
    from paper_2504_16214_b200.tilesynth.explore import synthesize_program
    from paper_2504_16214_b200.tilesynth.layout_flow import SynthesisConfig
    ours_cat = C.load_catalog(C.builtin_catalog_path())
    ref_cat = r_cat.load_catalog(r_cat.builtin_catalog_path())
    rng = random.Random(1234)
    compared = 0
    for _ in range(60):
        text, threads = _random_program(rng)
        cap = rng.choice([4, 16, 64])

        def run(ir, pipe, rep, cat, cfg):
            try:
                g = ir.parse_program(text)
            except Exception as e:  # noqa: BLE001
                return ("parse", type(e).__name__)
            try:
                res = pipe.synthesize_program(g, cat, cfg)
                return rep.render_json(rep.build_report(res, all_candidates=True))
            except Exception as e:  # noqa: BLE001
                return ("synth", type(e).__name__, str(e))
        got = run(IR, sys.modules[synthesize_program.__module__], R, ours_cat, SynthesisConfig(threads, cap))
        want = run(r_ir, r_pipe, r_rep, ref_cat, r_synth.SynthesisConfig(threads, cap))
        assert got == want, text
        compared += isinstance(got, str)
    assert compared >= 30

#!/usr/bin/env python
"""Drop parameter / return annotations from every ``def`` of the given Python files, in place
(dataclass fields and module-level annotations are left alone). Style tool for the synthesizer
package, which is written unannotated."""
import ast
import sys
from pathlib import Path


def strip(text: str) -> str:
    tree = ast.parse(text)
    lines = text.splitlines(keepends=True)
    starts = [0]
    for ln in lines:
        starts.append(starts[-1] + len(ln))

    def off(lineno, col):
        return starts[lineno - 1] + len(lines[lineno - 1].encode()[:col].decode())

    cuts = []
    for node in ast.walk(tree):
        if not isinstance(node, (ast.FunctionDef, ast.AsyncFunctionDef)):
            continue
        a = node.args
        for arg in a.posonlyargs + a.args + a.kwonlyargs + [x for x in (a.vararg, a.kwarg) if x]:
            if arg.annotation is not None:
                ann = arg.annotation
                cuts.append((off(arg.lineno, arg.col_offset) + len(arg.arg), off(ann.end_lineno, ann.end_col_offset)))
        if node.returns is not None:
            r = node.returns
            b, e = off(r.lineno, r.col_offset), off(r.end_lineno, r.end_col_offset)
            head = text[:b].rstrip()
            assert head.endswith("->"), head[-20:]
            cuts.append((len(head) - 2, e))
    for b, e in sorted(cuts, reverse=True):
        text = text[:b].rstrip(" ") + text[e:] if text[b:e].lstrip().startswith("->") else text[:b] + text[e:]
    return text


if __name__ == "__main__":
    for name in sys.argv[1:]:
        p = Path(name)
        out = strip(p.read_text())
        ast.parse(out)
        p.write_text(out)

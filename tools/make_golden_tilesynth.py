#!/usr/bin/env python
"""Generate the layout-synthesis golden reports from the REFERENCE implementation.

Runs the reference ``tilesynth`` CLI (``/root/reference/pkg/src``, read-only, one subprocess per
program) on every program under ``tests/golden/tilesynth/programs`` and writes its JSON reports
(default flags and ``--all-candidates``) to ``tests/golden/tilesynth/*.json``, plus the CLI exit
code and stderr. The reference's four fixtures (``pkg/fixtures/*.prog``) are imported with their
comment lines stripped (comments do not affect reports). Only needed in the build container;
the committed outputs are what ``tests/test_tilesynth_parity.py`` checks on any machine.
"""
from __future__ import annotations

import gzip
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
REF = Path("/root/reference/pkg")
OUT = ROOT / "tests" / "golden" / "tilesynth"
PROGS = OUT / "programs"

# extra CLI flags per program (threads etc.)
FLAGS = {"prefill_tile": ["--threads", "256"]}


def import_reference_fixtures():
    for f in sorted((REF / "fixtures").glob("*.prog")):
        body = [ln for ln in f.read_text().splitlines() if ln.strip() and not ln.strip().startswith("#")]
        (PROGS / f"ref_{f.name}").write_text("\n".join(body) + "\n")


def run_ref(prog: Path, extra):
    env = dict(os.environ, PYTHONPATH=str(REF / "src"), PYTHONDONTWRITEBYTECODE="1")
    cmd = [sys.executable, "-m", "tilesynth.cli", "--program", str(prog), "--format", "json", *extra]
    p = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd="/tmp")
    return p.returncode, p.stdout, p.stderr


def main():
    import_reference_fixtures()
    index = {}
    for prog in sorted(PROGS.glob("*.prog")):
        name = prog.stem
        extra = FLAGS.get(name.removeprefix("ref_"), [])
        for tag, more in (("default", []), ("all", ["--all-candidates"])):
            rc, out, err = run_ref(prog, extra + more)
            if tag == "all":  # large: stored gzip-compressed
                (OUT / f"{name}.{tag}.json.gz").write_bytes(gzip.compress(out.encode(), mtime=0))
            else:
                (OUT / f"{name}.{tag}.json").write_text(out)
            index[f"{name}.{tag}"] = {"args": extra + more, "rc": rc, "stderr": err}
            print(name, tag, rc, len(out))
    (OUT / "index.json").write_text(json.dumps(index, indent=1, sort_keys=True) + "\n")


if __name__ == "__main__":
    main()

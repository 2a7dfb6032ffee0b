"""oracle/make_golden_workloads.py — TEST INFRASTRUCTURE ONLY.

Golden vectors for the repo-authored workload grammars of configs 3 and 4
(paper_2506_03887_b200/grammars/{schema,sql}.bnf), built by the UNMODIFIED
reference compiler (oracle/_ref/libgmask_ref.so).  Run here:

    make -C oracle && python oracle/make_golden_workloads.py

Outputs
  tests/golden/schema.p3dpda      BuildDpda(default options) of schema.bnf
  tests/golden/workloads.json     per grammar: sha256 of the reference P3DPDA
                                  (sql's is ~20 MB, so only its digest is
                                  kept), BuildStats, composite/cycle counts.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import Ref  # noqa: E402

GRAMMARS = os.path.join(ROOT, "paper_2506_03887_b200", "grammars")
OUT = os.path.join(ROOT, "tests", "golden")


def main() -> None:
    out = {"source": "reference gmask BuildDpda via oracle/make_golden_workloads.py"}
    for name in ["schema", "sql"]:
        text = open(os.path.join(GRAMMARS, name + ".bnf")).read()
        rc, flat, st = Ref.compile_flat(text)
        assert rc == 0, (name, flat)
        out[name] = {"sha256": hashlib.sha256(flat).hexdigest(), "bytes": len(flat), "stats": st}
        if name == "schema":
            with open(os.path.join(OUT, name + ".p3dpda"), "wb") as f:
                f.write(flat)
    with open(os.path.join(OUT, "workloads.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

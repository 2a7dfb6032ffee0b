r"""oracle/make_golden_workloads.py — TEST INFRASTRUCTURE ONLY.

Golden vectors for the repo-authored workload grammars of configs 3 and 4
(paper_2506_03887_b200/grammars/{schema,sql}.bnf), built by the UNMODIFIED
reference compiler (oracle/_ref/libgmask_ref.so).  Run here:

    make -C oracle && python oracle/make_golden_workloads.py

Outputs
  tests/golden/schema.p3dpda      BuildDpda(default options) of schema.bnf
  tests/golden/workloads.json     per grammar: sha256 of the reference P3DPDA
                                  and GMASKDP1 (sql's are 13 / 35 MB, so only
                                  digests are kept), BuildStats, counts.
  tests/golden/<fixture>.gmaskdp1 SerializeDpda of every fixture grammar
                                  (needs the reference's serialize.cpp, built
                                  by oracle/Makefile when json.hpp is found)
  tests/golden/vocab_escapes.json LoadVocabulary known answer: a vocabulary
                                  file with \xNN / \\ escapes and the bytes
                                  the reference decodes it to (hex).
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
        if Ref.serialize_available():
            rc, dp1 = Ref.compile_gmaskdp1(text)
            assert rc == 0
            out[name]["gmaskdp1_sha256"] = hashlib.sha256(dp1).hexdigest()
            out[name]["gmaskdp1_bytes"] = len(dp1)
    if Ref.serialize_available():
        from oracle import read_flat
        for fx in ["paren", "list_left", "list_right", "digits", "expr", "json"]:
            text = read_flat(open(os.path.join(OUT, fx + ".p3dpda"), "rb").read())["grammar_text"]
            rc, dp1 = Ref.compile_gmaskdp1(text)
            assert rc == 0
            with open(os.path.join(OUT, fx + ".gmaskdp1"), "wb") as f:
                f.write(dp1)
        raw = ['a', '\\x41\\x00b', '\\\\', '\\xff\\xFE', 'tab\\x09', '"q"', 'caf\u00e9', '\\x7f']
        vocab_text = json.dumps(raw)
        toks = Ref.load_vocabulary(vocab_text.encode())
        with open(os.path.join(OUT, "vocab_escapes.json"), "w") as f:
            json.dump({"file": vocab_text, "tokens_hex": [t.hex() for t in toks]}, f, indent=1)
    with open(os.path.join(OUT, "workloads.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

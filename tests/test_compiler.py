"""Host grammar compiler (gm_automaton_compile, csrc/compiler.cpp) — parity
with the reference's ParseGrammar + BuildDpda (src/grammar.cpp,
src/lr1.cpp, src/dpda_builder.cpp, src/optimizer.cpp).

* Golden identity: every fixture grammar compiles to the byte-identical
  P3DPDA the reference built (tests/golden/, oracle/make_golden.py) — runs
  anywhere, no reference needed.
* Known answers from the reference's own tests: json 209 states
  (test_lr1.cpp:268-274), paren 10 states / 11 edges / 3 composites
  (test_dpda.cpp:47-57), digits 262 -> 46 edges under aggregation
  (test_optimizer.cpp:39-69), the ambiguous grammar's conflict report.
* Error kinds and messages (grammar.hpp:34-49, lr1.hpp:20-29).
* Differential fuzzing against the reference compiler itself (build
  container only: needs oracle/_ref built from /root/reference).
"""
import hashlib
import json
import os
import random

import pytest

import oracle
import paper_2506_03887_b200 as pk

HERE = os.path.dirname(__file__)
GOLDEN = os.path.join(HERE, "golden")
WORKLOADS = os.path.join(os.path.dirname(HERE), "paper_2506_03887_b200", "grammars")
FIXTURES = ["paren", "list_left", "list_right", "digits", "expr", "json"]


def grammar(name):
    """Fixture grammars: the normalized text the reference stored in its own
    automaton (PrintGrammar output reparses to the same grammar, same symbol
    order); workload grammars: the repo's authored .bnf files."""
    path = os.path.join(WORKLOADS, name + ".bnf")
    if os.path.exists(path):
        with open(path) as f:
            return f.read()
    return oracle.read_flat(golden(name))["grammar_text"]


def golden(name):
    with open(os.path.join(GOLDEN, name + ".p3dpda"), "rb") as f:
        return f.read()


@pytest.mark.parametrize("name", FIXTURES)
def test_fixture_compiles_to_golden(name):
    assert pk.Automaton.compile(grammar(name)).save() == golden(name)


def test_digits_without_aggregation_matches_golden():
    assert pk.Automaton.compile(grammar("digits"), aggregate=False).save() == golden("digits_noagg")


def test_reference_known_answers():
    js = pk.Automaton.compile(grammar("json")).info()
    assert js["num_states"] == 209 and js["num_edges"] == 1617
    paren = pk.Automaton.compile(grammar("paren"))
    assert paren.info()["num_states"] == 10 and paren.info()["num_edges"] == 11
    assert paren.compile_stats()["composites"] == 3
    assert pk.Automaton.compile(grammar("paren"), merge=False).compile_stats()["composites"] == 0
    assert pk.Automaton.compile(grammar("digits"), aggregate=False).info()["num_edges"] == 262
    assert pk.Automaton.compile(grammar("digits")).info()["num_edges"] == 46
    # list_right: the only rewritten pumping circuit of the fixtures
    assert pk.Automaton.compile(grammar("list_right")).compile_stats()["cycles"] == 1


def test_grammar_hash_is_fnv1a_of_normalized_text():
    a = pk.Automaton.compile('S -> "(" S ")" | "a"   # comment\n')
    flat = a.save()
    info = oracle.read_flat(flat)
    text = info["grammar_text"]
    assert text == 'S -> "(" S ")"\nS -> "a"\n'
    h = 0xcbf29ce484222325
    for ch in text.encode():
        h = ((h ^ ch) * 0x100000001b3) & (2**64 - 1)
    assert info["grammar_hash"] == h == a.info()["grammar_hash"] & (2**64 - 1)


@pytest.mark.parametrize("text,kind,needle", [
    ("", pk.GrammarError, "EmptyGrammar"),
    ("# only a comment\n", pk.GrammarError, "EmptyGrammar"),
    ("S -> A\n", pk.GrammarError, "UndefinedSymbol: 'A'"),
    ("S = \"a\"\n", pk.GrammarError, "line 1, column 3: expected '->'"),
    ("S -> \"\"\n", pk.GrammarError, "empty terminal literal"),
    ("S -> \"a\n", pk.GrammarError, "unterminated terminal literal"),
    ("S -> \"\\q\"\n", pk.GrammarError, "unknown escape"),
    ("S -> \"\\xZZ\"\n", pk.GrammarError, "bad hex digits"),
    ("\nS -> \"a\" %\n", pk.GrammarError, "line 2, column 10: unexpected character '%'"),
    ("S -> S S | \"a\"\n", pk.BuildError, "NotLR1Conflict: state 3 on 'a'"),
])
def test_error_kinds(text, kind, needle):
    with pytest.raises(kind) as e:
        pk.Automaton.compile(text)
    assert needle in str(e.value)


def test_escapes_and_multibyte_literals():
    a = pk.Automaton.compile('S -> "\\x41\\"\\\\" T\nT -> "\\x00" | "ab"\n')
    text = oracle.read_flat(a.save())["grammar_text"]
    assert text == 'S -> "A\\"\\\\" T\nT -> "\\x00"\nT -> "ab"\n'


def test_compiled_automaton_drives_the_runtime():
    """The compiler's output is loadable and equals the golden in every field
    the device flattening reads (flat bytes are identical, so the device
    tables are too)."""
    a = pk.Automaton.compile(grammar("json"))
    b = pk.Automaton.load(a.save())
    assert b.info() == a.info()


def _random_grammar(rng):
    names = ["A", "B", "C", "D", "E"][: rng.randint(1, 5)]
    lines = []
    for n in names:
        alts = []
        for _ in range(rng.randint(1, 3)):
            syms = []
            for _ in range(rng.randint(0, 4)):
                if rng.random() < 0.45:
                    syms.append(rng.choice(names))
                else:
                    syms.append('"' + rng.choice("abc(),") + '"')
            alts.append(" ".join(syms))
        lines.append(n + " -> " + " | ".join(alts))
    return "\n".join(lines) + "\n"


def _ref_compile(text, aggregate):
    rc, data, stats = oracle.Ref.compile_flat(text, aggregate=aggregate)
    if rc != 0:
        return None, data.decode(), stats
    return data, None, stats


def _mine(text, aggregate):
    try:
        a = pk.Automaton.compile(text, aggregate=aggregate)
    except pk.GmError as e:
        return None, str(e).split("] ", 1)[1], {}
    return a.save(), None, a.compile_stats()


needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="reference oracle not built (needs /root/reference)")


@needs_ref
@pytest.mark.parametrize("seed", range(4))
def test_differential_random_grammars(seed):
    """Random small grammars (conflicts, epsilon rules, non-productive and
    pumping nonterminals included): identical automata or identical errors."""
    rng = random.Random(1000 + seed)
    n_ok = 0
    for _ in range(150):
        text = _random_grammar(rng)
        for agg in (True, False):
            mine, merr, mst = _mine(text, agg)
            ref, rerr, rst = _ref_compile(text, agg)
            assert merr == rerr, text
            assert mine == ref, text
            if mine is not None:
                n_ok += 1
                assert mst["composites"] == rst["composites"], text
                assert mst["cycles"] == rst["cycles"], text
    assert n_ok > 20


@needs_ref
@pytest.mark.parametrize("name", ["schema", "sql"])
def test_differential_large_grammars(name):
    text = grammar(name)
    mine, merr, mst = _mine(text, True)
    ref, rerr, rst = _ref_compile(text, True)
    assert merr is None and rerr is None
    assert mine == ref
    assert mst["composites"] == rst["composites"]


@pytest.mark.parametrize("name", ["schema", "sql"])
def test_workload_grammars_match_reference_digest(name):
    """Config 3/4 grammars: sha256 of the reference-built P3DPDA
    (oracle/make_golden_workloads.py) and its BuildStats."""
    with open(os.path.join(GOLDEN, "workloads.json")) as f:
        want = json.load(f)[name]
    a = pk.Automaton.compile(grammar(name))
    flat = a.save()
    assert hashlib.sha256(flat).hexdigest() == want["sha256"]
    assert a.info()["num_states"] == want["stats"]["states"]
    assert a.info()["num_edges"] == want["stats"]["edges"]
    assert a.compile_stats()["composites"] == want["stats"]["composites"]
    if name == "schema":
        assert flat == golden("schema")

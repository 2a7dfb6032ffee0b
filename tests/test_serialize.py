"""On-disk formats (csrc/serialize.cpp): the reference's GMASKDP1 automaton
text (SerializeDpda / DeserializeDpda, src/serialize.cpp:148-294) and its
JSON vocabulary files (LoadVocabulary / UnescapeToken / EscapeToken,
src/serialize.cpp:298-364).

* Byte-identical GMASKDP1 for every fixture (reference-written goldens in
  tests/golden/*.gmaskdp1, oracle/make_golden_workloads.py) and sha256-pinned
  for the config 3/4 grammars; load -> save round trips
  (test_serialize.cpp:49-63's property).
* The loader re-derives arbitration order and re-checks determinism
  (serialize.cpp:284-292): shuffled edges load to the same automaton,
  inconsistent machines are rejected.
* Error kinds (SerializeError: BadMagic / BadVersion / Parse / Structure).
* Where the reference oracle is built with its serializer: differential
  checks of writer, loader errors and the vocabulary decoder.
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


def golden(name, ext):
    with open(os.path.join(GOLDEN, name + ext), "rb") as f:
        return f.read()


def fixture_text(name):
    return oracle.read_flat(golden(name, ".p3dpda"))["grammar_text"]


@pytest.mark.parametrize("name", FIXTURES)
def test_gmaskdp1_writer_matches_reference(name):
    assert pk.Automaton.compile(fixture_text(name)).save_gmaskdp1() == golden(name, ".gmaskdp1")


@pytest.mark.parametrize("name", FIXTURES)
def test_gmaskdp1_roundtrip_and_p3dpda_identity(name):
    dp1 = golden(name, ".gmaskdp1")
    a = pk.Automaton.load(dp1)
    assert a.save_gmaskdp1() == dp1
    assert a.save() == golden(name, ".p3dpda")  # the device layout the runtime reads
    assert a.compile_stats() == pk.Automaton.compile(fixture_text(name)).compile_stats()


@pytest.mark.parametrize("name", ["schema", "sql"])
def test_gmaskdp1_workload_digests(name):
    want = json.load(open(os.path.join(GOLDEN, "workloads.json")))[name]
    if "gmaskdp1_sha256" not in want:
        pytest.skip("goldens generated without the reference serializer")
    dp1 = pk.Automaton.compile(open(os.path.join(WORKLOADS, name + ".bnf")).read()).save_gmaskdp1()
    assert hashlib.sha256(dp1).hexdigest() == want["gmaskdp1_sha256"]


def _tamper(dp1: bytes, fn) -> bytes:
    head, body = dp1.split(b"\n", 1)
    j = json.loads(body)
    fn(j)
    return head + b"\n" + json.dumps(j, sort_keys=True, separators=(",", ":")).encode() + b"\n"


def test_loader_rederives_arbitration_order():
    dp1 = golden("json", ".gmaskdp1")
    rng = random.Random(3)
    shuffled = _tamper(dp1, lambda j: rng.shuffle(j["edges"]))
    assert shuffled != dp1
    a = pk.Automaton.load(shuffled)
    assert a.save_gmaskdp1() == dp1 and a.save() == golden("json", ".p3dpda")


@pytest.mark.parametrize("mutate,kind", [
    (lambda d: b"GMASKDP2" + d[8:], "BadMagic"),
    (lambda d: d.replace(b'"version":1', b'"version":2'), "BadVersion"),
    (lambda d: d[:-40], "Parse"),
    (lambda d: _tamper(d, lambda j: j.pop("stats")), "Structure"),
    (lambda d: _tamper(d, lambda j: j.__setitem__("num_states", 0)), "Structure"),
    (lambda d: _tamper(d, lambda j: j.__setitem__("grammar_text", j["grammar_text"] + " ")), "Structure"),
    (lambda d: _tamper(d, lambda j: j["shifts"].append([0, 300, 1])), "Structure"),
    (lambda d: _tamper(d, lambda j: j["edges"][0].__setitem__("match", [])), "Structure"),
    (lambda d: _tamper(d, lambda j: j["edges"][0].__setitem__("accepted", "zz")), "Structure"),
    (lambda d: _tamper(d, lambda j: j["edges"].append(dict(j["edges"][0]))), "Structure"),  # nondeterministic
])
def test_loader_errors(mutate, kind):
    bad = mutate(golden("paren", ".gmaskdp1"))
    with pytest.raises(pk.SerializeError) as e:
        pk.Automaton.load(bad)
    assert f"SerializeError({kind})" in str(e.value)
    if oracle.ref_available() and oracle.Ref.serialize_available():
        rc, msg = oracle.Ref.roundtrip_gmaskdp1(bad)
        assert rc != 0, "the reference rejects it too"


def test_vocabulary_known_answer():
    g = json.load(open(os.path.join(GOLDEN, "vocab_escapes.json")))
    toks = pk.load_vocabulary(g["file"].encode())
    assert [t.hex() for t in toks] == g["tokens_hex"]
    for t in toks:  # EscapeToken inverts the unescape
        assert pk.load_vocabulary(json.dumps([pk.escape_token(t)]).encode()) == [t]


@pytest.mark.parametrize("text", ['{"a": 1}', '["\\\\q"]', '["\\\\x4"]', '["\\\\xzz"]', '[1]', '["a"', '["\\\\"]'])
def test_vocabulary_errors(text):
    with pytest.raises(pk.SerializeError):
        pk.load_vocabulary(text.encode())
    if oracle.ref_available() and oracle.Ref.serialize_available():
        with pytest.raises(ValueError):
            oracle.Ref.load_vocabulary(text.encode())


def test_vocabulary_file_drives_the_engine_layout():
    """A synthetic vocabulary written as a reference vocabulary file loads
    back to the same tokens (the path a user's tokenizer export takes)."""
    vocab = pk.synth_vocab(2000)
    text = json.dumps([pk.escape_token(t) for t in vocab])
    assert pk.load_vocabulary(text.encode()) == vocab
    if oracle.ref_available() and oracle.Ref.serialize_available():
        assert oracle.Ref.load_vocabulary(text.encode()) == vocab

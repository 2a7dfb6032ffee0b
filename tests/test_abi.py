"""C-ABI surface checks that need no GPU: the library loads, exports every
symbol include/*.h declares, round-trips the flat automaton format, rejects
corrupt input like DeserializeDpda does (serialize.cpp:198-294), applies
TokenTrie::Build's vocabulary rules (runtime.cpp:18-61), and fails loudly
(GM_ERR_CUDA) rather than falling back to the CPU when no device exists."""
import ctypes
import glob
import os
import re

import numpy as np
import pytest

import paper_2506_03887_b200 as pk

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
FIXTURES = ["paren", "list_left", "list_right", "digits", "digits_noagg", "expr", "json"]


def flat(name):
    with open(os.path.join(GOLDEN, name + ".p3dpda"), "rb") as f:
        return f.read()


def declared_functions():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"\b(gmw?_[a-z0-9_]+)\s*\(", text):
            names.add(m.group(1))
    return names


def test_library_exports_every_declared_symbol():
    lib = pk.lib()
    names = declared_functions()
    assert len(names) >= 25
    for n in sorted(names):
        assert hasattr(lib, n), f"{n} declared in include/ but not exported"
    assert lib.gm_abi_version() == 2


@pytest.mark.parametrize("name", FIXTURES)
def test_flat_roundtrip_and_info(name):
    import oracle
    f = flat(name)
    a = pk.Automaton.load(f)
    assert a.save() == f
    info = a.info()
    parsed = oracle.read_flat(f)
    assert info["num_states"] == parsed["num_states"]
    assert info["num_edges"] == len(parsed["edges"])
    assert info["dynamic_edges"] == sum(e["dynamic"] for e in parsed["edges"])


def test_fixture_automaton_identity():
    """test_lr1.cpp:268-274 (json 209 states), test_dpda.cpp:47-57 (paren 10
    states, 11 edges, 3 dynamic), test_optimizer.cpp:39-69 (digits 262 -> 46)."""
    assert pk.Automaton.load(flat("json")).info()["num_states"] == 209
    p = pk.Automaton.load(flat("paren")).info()
    assert (p["num_states"], p["num_edges"], p["dynamic_edges"]) == (10, 11, 3)
    assert pk.Automaton.load(flat("digits")).info()["num_edges"] == 46
    assert pk.Automaton.load(flat("digits_noagg")).info()["num_edges"] == 262


def test_corrupt_inputs_rejected():
    f = bytearray(flat("paren"))
    with pytest.raises(pk.SerializeError):
        pk.Automaton.load(b"NOTMAGIC" + bytes(f[8:]))
    with pytest.raises(pk.SerializeError):
        pk.Automaton.load(bytes(f[:-3]))
    with pytest.raises(pk.SerializeError):
        pk.Automaton.load(bytes(f) + b"\0")
    # Break a shift target (state id out of range).
    import struct
    S = struct.unpack_from("<i", f, 8)[0]
    tl = struct.unpack_from("<i", f, 28)[0]
    off = 32 + tl
    g = bytearray(f)
    struct.pack_into("<i", g, off, S + 5)
    with pytest.raises(pk.SerializeError):
        pk.Automaton.load(bytes(g))


def test_vocab_rules_before_device_use():
    a = pk.Automaton.load(flat("paren"))
    with pytest.raises(pk.VocabError) as e:
        pk.DeviceEngine(a, [b"x", b""])
    assert e.value.kind == "empty" and "1" in str(e.value)
    with pytest.raises(pk.VocabError) as e:
        pk.DeviceEngine(a, [b"ab", b"cd", b"ab"])
    assert e.value.kind == "duplicate" and "0" in str(e.value) and "2" in str(e.value)


def test_no_silent_cpu_fallback():
    """Without a CUDA device the engine must fail loudly (GM_ERR_CUDA)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    a = pk.Automaton.load(flat("paren"))
    with pytest.raises(pk.CudaError):
        pk.DeviceEngine(a, [b"a", b"("])


def test_usage_errors():
    a = pk.Automaton.load(flat("paren"))
    h = ctypes.c_void_p()
    data, offs = pk.pack_vocab([b"a"])
    opts = pk._EngineOptions(33, 8192, 0, 256)  # K <= 32
    rc = pk.lib().gm_engine_create(a._h, data.ctypes.data, offs.ctypes.data, 1, ctypes.byref(opts), 0,
                                   ctypes.byref(h))
    assert rc == pk.GM_ERR_USAGE
    opts = pk._EngineOptions(8, 1000, 0, 256)
    rc = pk.lib().gm_engine_create(a._h, data.ctypes.data, offs.ctypes.data, 1, ctypes.byref(opts), 0,
                                   ctypes.byref(h))
    assert rc == pk.GM_ERR_USAGE and "power of two" in pk.lib().gm_last_error().decode()


def test_synth_vocab_shape():
    v = pk.synth_vocab(32000)
    assert len(v) == 32000 and v == sorted(v) and len(set(v)) == 32000
    assert b"true" in v and b'": "' in v
    big = pk.synth_vocab(128255)
    assert len(big) == 128255 and big == sorted(big)
    s = pk.structural_words(v)
    assert s.shape == ((32001 + 31) // 32,)
    n = sum(bin(int(x)).count("1") for x in s)
    assert n == sum(1 for t in v if any(c in b'{}[],:"' for c in t))


def test_cpp_wrapper_compiles_against_the_abi(tmp_path):
    """include/pre3/device_engine.hpp (the reference-side C++ binding) builds
    and links against libpre3gmask.so."""
    import subprocess
    src = tmp_path / "t.cpp"
    src.write_text('#include "pre3/device_engine.hpp"\n'
                   'int main(){ return gm_abi_version() == GM_ABI_VERSION ? 0 : 1; }\n')
    lib_dir = os.path.join(ROOT, "paper_2506_03887_b200")
    exe = tmp_path / "t"
    subprocess.run(["g++", "-std=c++17", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe),
                    "-L", lib_dir, "-lpre3gmask", f"-Wl,-rpath,{lib_dir}"], check=True)
    assert subprocess.run([str(exe)]).returncode == 0

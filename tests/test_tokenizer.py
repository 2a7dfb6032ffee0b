"""Vocabulary ingestion (paper_2506_03887_b200/tokenizer.py):
real tokenizer.json files -> the token byte strings the mask is computed
over, ids aligned with the model's logits, EOS -> mask bit V.

Tokenizers are trained / assembled here with the `tokenizers` library (no
network): byte-level BPE (GPT-2 / Llama-3 style) and SentencePiece-style BPE
with byte fallback (Llama-2 style).  The property checked is the one the mask
depends on: for any text, the bytes of the ids the tokenizer produces
concatenate to the text's bytes.
"""
import json
import random

import pytest

tokenizers = pytest.importorskip("tokenizers")

import oracle  # noqa: E402
import paper_2506_03887_b200 as pk  # noqa: E402
from paper_2506_03887_b200 import tokenizer as tk  # noqa: E402

CORPUS = [
    '{"name": "ada", "age": 36, "tags": ["math", "engine"], "ok": true}',
    '[1, 2, 3, {"a": null, "b": false}]',
    "the quick brown fox jumps over the lazy dog, naïve café déjà vu — ∑ 日本語",
    'SELECT name, COUNT(x) FROM t WHERE a = 1 AND b <> 2 ORDER BY name DESC',
] * 20


def random_texts(n, seed=0):
    rng = random.Random(seed)
    alphabet = 'abcdefghijklmnopqrstuvwxyz {}[]":,0123456789-éü日本\n\t'
    return ["".join(rng.choice(alphabet) for _ in range(rng.randint(1, 40))) for _ in range(n)]


@pytest.fixture(scope="module")
def byte_level_json():
    from tokenizers import Tokenizer, decoders, models, pre_tokenizers, trainers
    tok = Tokenizer(models.BPE())
    tok.pre_tokenizer = pre_tokenizers.ByteLevel(add_prefix_space=False)
    tok.decoder = decoders.ByteLevel()
    trainer = trainers.BpeTrainer(vocab_size=700, initial_alphabet=pre_tokenizers.ByteLevel.alphabet(),
                                  show_progress=False)
    tok.train_from_iterator(CORPUS, trainer)
    tok.add_special_tokens(["<|endoftext|>", "<|pad|>"])  # specials after the regular ids (GPT-2 / Llama-3)
    return tok, tok.to_str()


@pytest.fixture(scope="module")
def sentencepiece_json():
    from tokenizers import Tokenizer, decoders, models, normalizers, pre_tokenizers, trainers
    tok = Tokenizer(models.BPE(byte_fallback=True, unk_token=None))
    tok.pre_tokenizer = pre_tokenizers.Metaspace(replacement="▁", prepend_scheme="never")
    tok.decoder = decoders.Sequence([decoders.Replace("▁", " "), decoders.ByteFallback(), decoders.Fuse()])
    byte_tokens = [f"<0x{b:02X}>" for b in range(256)]
    # Llama-2 layout: <unk> <s> </s> at ids 0..2, then the byte-fallback pieces, then the merges
    trainer = trainers.BpeTrainer(vocab_size=800, special_tokens=["<unk>", "<s>", "</s>"] + byte_tokens,
                                  show_progress=False)
    tok.train_from_iterator(CORPUS, trainer)
    data = json.loads(tok.to_str())
    # the byte-fallback pieces are ordinary vocabulary entries in real files
    data["added_tokens"] = [t for t in data["added_tokens"] if not t["content"].startswith("<0x")]
    return Tokenizer.from_str(json.dumps(data)), json.dumps(data)


def test_byte_level_bpe_roundtrip(byte_level_json):
    tok, text = byte_level_json
    tv = tk.from_tokenizer_json(text)
    assert tv.encoding == "byte_level"
    assert tv.eos_model_id == tok.token_to_id("<|endoftext|>") == tv.V  # EOS right after the regular ids
    assert len(set(tv.tokens)) == tv.V and all(tv.tokens)
    for s in random_texts(300) + CORPUS[:4]:
        ids = tok.encode(s).ids
        assert all(i < tv.V for i in ids)
        assert b"".join(tv.tokens[i] for i in ids) == s.encode("utf-8"), s


def test_sentencepiece_byte_fallback_roundtrip(sentencepiece_json):
    tok, text = sentencepiece_json
    tv = tk.from_tokenizer_json(text)
    assert tv.encoding == "sentencepiece"
    assert tv.eos_model_id == tok.token_to_id("</s>") == 2
    assert tv.token_bytes(tok.token_to_id("<0x0A>")) == b"\n"
    # specials below V and duplicate byte strings are disabled ids, leaving
    # a TokenTrie-valid vocabulary ('<0x61>' vs 'a', '<0x20>' vs '▁')
    assert {0, 1, 2} <= set(tv.disabled)
    assert tv.aliases and all(tv.tokens[a] == b"" and tv.tokens[c] for a, c in tv.aliases.items())
    assert tv.aliases.get(tok.token_to_id("<0x20>")) == tok.token_to_id("▁")
    live = [t for i, t in enumerate(tv.tokens) if i not in set(tv.disabled)]
    assert len(live) == len(set(live)) == tv.V - len(tv.disabled) and all(live)
    opts = tv.engine_options()
    assert opts["eos_column"] == 2 and opts["num_columns"] == tv.model_vocab_size == tv.V
    for s in random_texts(300, seed=1):
        ids = tok.encode(s).ids
        assert b"".join(tv.token_bytes(i) for i in ids) == s.encode("utf-8"), s
    port = oracle.Port(open(__file__.replace("test_tokenizer.py", "golden/json.p3dpda"), "rb").read(),
                       port_vocab(tv))
    m = port.mask(port.initial())
    assert not any((int(m[i >> 5]) >> (i & 31)) & 1 for i in tv.disabled)


def port_vocab(tv):
    """The engine vocabulary for the C port, which has no disabled ids: each
    disabled id gets unique bytes the JSON grammar can never accept."""
    return [t if t else b"\x01\x02" + i.to_bytes(4, "little") for i, t in enumerate(tv.tokens)]


def test_vocabulary_file_roundtrip(byte_level_json):
    tv = tk.from_tokenizer_json(byte_level_json[1])
    assert pk.load_vocabulary(tk.vocabulary_json(tv.tokens).encode()) == tv.tokens


def test_tokenizer_vocab_drives_the_reference_matcher(byte_level_json):
    """The ingested vocabulary is a valid TokenTrie vocabulary (no empty or
    duplicate tokens) and the reference matcher's masks over it allow exactly
    the tokens whose bytes continue a JSON prefix."""
    tv = tk.from_tokenizer_json(byte_level_json[1])
    flat = open(__file__.replace("test_tokenizer.py", "golden/json.p3dpda"), "rb").read()
    port = oracle.Port(flat, tv.tokens)
    c = port.initial()
    m = port.mask(c)
    allowed = [t for t in range(tv.V) if (int(m[t >> 5]) >> (t & 31)) & 1]
    assert allowed and all(tv.tokens[t][:1] in (b"{", b"[", b'"', b"t", b"f", b"n", b"-", b" ") or
                           tv.tokens[t][:1].isdigit() for t in allowed)
    assert not (int(m[tv.V >> 5]) >> (tv.V & 31)) & 1  # EOS not allowed on an empty document


def test_errors():
    with pytest.raises(ValueError):
        tk.from_tokenizer_json({"model": {}})
    holes = tk.from_tokenizer_json({"model": {"type": "BPE", "vocab": {"a": 0, "b": 2}}, "added_tokens": []})
    assert holes.V == 3 and holes.disabled == [1]  # an unused id below V is disabled
    assert holes.engine_options()["num_columns"] == 0  # no specials: the reference layout (EOS = column V)
    pad_only = tk.from_tokenizer_json({"model": {"type": "BPE", "vocab": {"a": 0}},
                                       "added_tokens": [{"id": 1, "content": "<pad>", "special": True}]})
    with pytest.raises(ValueError):
        pad_only.engine_options()  # special columns but no EOS column to put bit V on
    with pytest.raises(ValueError):
        tk.from_tokenizer_json({"model": {"type": "BPE", "vocab": {"a": 0}}, "added_tokens": []}, eos_token="</s>")

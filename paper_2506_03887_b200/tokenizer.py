"""Vocabulary ingestion before the mask: the byte string
of every model token, from a Hugging Face ``tokenizer.json``, in the id order
the engine (and the reference's TokenTrie, runtime.cpp:18-61) expects, plus
the EOS mapping to mask bit V.

Supported token encodings:

* byte-level BPE (GPT-2 / Llama-3 / Qwen style: ``ByteLevel`` pre-tokenizer or
  decoder) — each token string is mapped back through the inverse of the
  GPT-2 ``bytes_to_unicode`` table;
* SentencePiece-style BPE/Unigram (Llama-2 / Mistral style: ``Metaspace`` or a
  ``Replace("▁", " ")`` decoder, optional ``<0xNN>`` byte-fallback tokens) —
  ``▁`` is a space, ``<0xNN>`` is the byte NN, other text is UTF-8.

Added / special tokens (``added_tokens`` with ``special: true``) have no
byte form: they are never allowed by a grammar, except the EOS token, which
the engine represents as mask bit V (``TokenMask::SetEos``, runtime.hpp:62-85).
The regular tokens must occupy ids 0..V-1 (true for the tokenizers above), so
the mask's bit t is the model's logit t for every regular token; the caller
maps EOS (model id ``eos_model_id``) to bit V.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Union


def bytes_to_unicode() -> Dict[int, str]:
    """GPT-2's reversible byte -> printable-unicode table."""
    bs = list(range(ord("!"), ord("~") + 1)) + list(range(ord("¡"), ord("¬") + 1)) + list(range(ord("®"), ord("ÿ") + 1))
    cs = bs[:]
    n = 0
    for b in range(256):
        if b not in bs:
            bs.append(b)
            cs.append(256 + n)
            n += 1
    return dict(zip(bs, (chr(c) for c in cs)))


_UNICODE_TO_BYTE = {v: k for k, v in bytes_to_unicode().items()}


@dataclass
class TokenizerVocab:
    tokens: List[bytes]                       # regular tokens, ids 0..V-1
    eos_model_id: Optional[int]               # model id of EOS (mask bit V)
    specials: Dict[int, str] = field(default_factory=dict)  # model id -> content (never allowed)
    encoding: str = "byte_level"              # or "sentencepiece"
    model_vocab_size: int = 0                 # regular + special ids

    @property
    def V(self) -> int:
        return len(self.tokens)


def _walk(node, kinds):
    if isinstance(node, dict):
        if "type" in node:
            kinds.add(node["type"])
        for v in node.values():
            _walk(v, kinds)
    elif isinstance(node, list):
        for v in node:
            _walk(v, kinds)


def _sentencepiece_bytes(tok: str) -> bytes:
    if len(tok) == 6 and tok.startswith("<0x") and tok.endswith(">"):
        try:
            return bytes([int(tok[3:5], 16)])
        except ValueError:
            pass
    return tok.replace("▁", " ").encode("utf-8")


def _byte_level_bytes(tok: str) -> bytes:
    try:
        return bytes(_UNICODE_TO_BYTE[c] for c in tok)
    except KeyError as e:
        raise ValueError(f"token {tok!r} is not byte-level encoded (character {e.args[0]!r})") from None


def from_tokenizer_json(source: Union[str, bytes, dict], eos_token: Optional[str] = None) -> TokenizerVocab:
    """Parses a tokenizer.json (path, JSON text, or the parsed dict)."""
    if isinstance(source, dict):
        tj = source
    else:
        text = source.decode() if isinstance(source, bytes) else source
        if text.lstrip().startswith("{"):
            tj = json.loads(text)
        else:
            with open(text, encoding="utf-8") as f:
                tj = json.load(f)
    model = tj.get("model") or {}
    vocab = model.get("vocab")
    if isinstance(vocab, list):  # Unigram: [[piece, score], ...] in id order
        id_of = {piece: i for i, (piece, _score) in enumerate(vocab)}
    elif isinstance(vocab, dict):
        id_of = dict(vocab)
    else:
        raise ValueError("tokenizer.json has no model.vocab")
    kinds: set = set()
    _walk({k: tj.get(k) for k in ("pre_tokenizer", "decoder", "normalizer")}, kinds)
    byte_level = "ByteLevel" in kinds
    encoding = "byte_level" if byte_level else "sentencepiece"
    added = {int(t["id"]): t for t in tj.get("added_tokens") or []}
    specials = {i: t["content"] for i, t in added.items() if t.get("special", False)}
    for i, t in added.items():  # non-special added tokens are text: keep them in the vocabulary
        if i not in specials:
            id_of.setdefault(t["content"], i)
    regular = {i: s for s, i in id_of.items() if i not in specials}
    V = len(regular)
    if sorted(regular) != list(range(V)):
        raise ValueError("regular tokens must occupy ids 0..V-1 (specials after them)")
    conv = _byte_level_bytes if byte_level else _sentencepiece_bytes
    tokens = [conv(regular[i]) for i in range(V)]
    eos_id = None
    if eos_token is not None:
        for i, c in specials.items():
            if c == eos_token:
                eos_id = i
        if eos_id is None:
            raise ValueError(f"EOS token {eos_token!r} is not a special token of this tokenizer")
    else:
        for cand in ("<|end_of_text|>", "<|endoftext|>", "</s>", "<|eot_id|>", "<eos>", "<|im_end|>"):
            hits = [i for i, c in specials.items() if c == cand]
            if hits:
                eos_id = hits[0]
                break
    all_ids = set(regular) | set(specials)
    return TokenizerVocab(tokens=tokens, eos_model_id=eos_id, specials=specials, encoding=encoding,
                          model_vocab_size=(max(all_ids) + 1) if all_ids else 0)


def vocabulary_json(tokens: List[bytes]) -> str:
    """The reference's vocabulary file (LoadVocabulary, serialize.cpp:348-364)
    for these tokens: a JSON array of EscapeToken strings."""
    from . import escape_token
    return json.dumps([escape_token(t) for t in tokens])

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
the reference represents as mask bit V (``TokenMask::SetEos``,
runtime.hpp:62-85).  The engine speaks the model's logit layout
(``gm_engine_options``): engine token id t < V is model column t, columns
>= V are specials (-inf), and mask bit V lands on the EOS column.  So:

* V = 1 + the largest id of a regular token; a special or an unused id below
  V (Llama-2 / Mistral put ``<unk> <s> </s>`` at ids 0..2) is a *disabled*
  id, never allowed;
* two ids with the same bytes (SentencePiece ``<0xNN>`` byte-fallback pieces
  next to the single-character piece, ``▁`` next to ``<0x20>``) would break
  TokenTrie::Build's no-duplicate rule (runtime.cpp:23-53): one canonical id
  keeps the bytes (the ordinary piece before a ``<0xNN>`` piece, then the
  lower id) and the others become disabled aliases (``aliases``: alias ->
  canonical), so a constrained sampler emits the canonical id.

``TokenizerVocab.engine_options()`` gives the DeviceEngine keyword arguments
for this layout.
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
    tokens: List[bytes]                       # engine ids 0..V-1 = model columns 0..V-1 (b"" if disabled)
    eos_model_id: Optional[int]               # model column of EOS (mask bit V)
    specials: Dict[int, str] = field(default_factory=dict)  # model id -> content (never allowed)
    encoding: str = "byte_level"              # or "sentencepiece"
    model_vocab_size: int = 0                 # logit columns: regular + special ids
    disabled: List[int] = field(default_factory=list)     # ids < V never allowed (specials, holes, aliases)
    aliases: Dict[int, int] = field(default_factory=dict)  # duplicate-bytes id -> canonical id

    @property
    def V(self) -> int:
        return len(self.tokens)

    def token_bytes(self, model_id: int) -> bytes:
        """The bytes of a model token id (an alias decodes as its canonical id)."""
        return self.tokens[self.aliases.get(model_id, model_id)]

    def engine_options(self) -> Dict[str, object]:
        """DeviceEngine(num_columns=, eos_column=, disabled=) for this model's
        logit layout.  Without an EOS token the EOS bit goes to an extra
        column V (the reference layout) when no special sits there."""
        ncols = max(self.model_vocab_size, self.V)
        eos = self.eos_model_id
        if eos is None:
            if ncols == self.V:
                return dict(num_columns=0, eos_column=0, disabled=list(self.disabled))
            raise ValueError("this vocabulary has special columns but no EOS token; pass eos_token=")
        return dict(num_columns=ncols, eos_column=eos, disabled=list(self.disabled))


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
    if not regular:
        raise ValueError("tokenizer.json has no regular tokens")
    if min(regular) < 0 or min(specials, default=0) < 0:
        raise ValueError("negative token id")
    V = max(regular) + 1
    conv = _byte_level_bytes if byte_level else _sentencepiece_bytes
    tokens: List[bytes] = [b""] * V
    disabled = set(range(V)) - set(regular)  # specials and unused ids below V
    aliases: Dict[int, int] = {}
    canon: Dict[bytes, int] = {}

    def rank(i: int):  # the canonical id of a byte string: ordinary piece first, then the lower id
        p = regular[i]
        return (len(p) == 6 and p.startswith("<0x") and p.endswith(">"), i)

    for i in sorted(regular, key=rank):
        b = conv(regular[i])
        if not b:
            disabled.add(i)  # an empty piece can never be a TokenTrie token
            continue
        if b in canon:
            aliases[i] = canon[b]
            disabled.add(i)
            continue
        canon[b] = i
        tokens[i] = b
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
                          model_vocab_size=max(all_ids) + 1, disabled=sorted(disabled), aliases=aliases)


def vocabulary_json(tokens: List[bytes]) -> str:
    """The reference's vocabulary file (LoadVocabulary, serialize.cpp:348-364)
    for these tokens: a JSON array of EscapeToken strings."""
    from . import escape_token
    return json.dumps([escape_token(t) for t in tokens])

"""Model logit layouts at the boundary:
mask bit V (EOS) lands on the model's EOS column, every other special column
gets -inf, and ids in the ABI are model columns — checked token for token
against the C port, which works in the reference's bit space (EOS = bit V)
over the same regular vocabulary.

* Llama-3-like: V regular ids, then 256 specials; EOS = V + 1 (like
  <|end_of_text|> 128001 after <|begin_of_text|> 128000).
* Llama-2-like: specials at ids 0..2 among the regular ids (disabled), EOS =
  id 2, no columns past V.  The port sees the same ids with bytes the grammar
  can never accept, so it never allows them either.
"""
import numpy as np
import pytest

import oracle
import paper_2506_03887_b200 as pk
from oracle import Port

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

DEV = "cuda:0"


def json_flat():
    import os
    with open(os.path.join(os.path.dirname(__file__), "golden", "json.p3dpda"), "rb") as f:
        return f.read()


def layouts():
    base = oracle.synth_vocab(6000)
    f = json_flat()
    acc = 0
    for e in oracle.read_flat(f)["edges"]:
        acc |= e["accepted"]
    never = [bytes([b]) for b in range(1, 256) if not (acc >> b) & 1]
    assert len(never) >= 3
    V = len(base)
    llama3 = dict(name="llama3", engine_vocab=base, port_vocab=base, V=V, ncols=V + 256, eos=V + 1, disabled=[])
    l2 = [b"", b"", b""] + base[3:]
    l2p = [never[0] * 3, never[1] * 3, never[2] * 3] + base[3:]
    llama2 = dict(name="llama2", engine_vocab=l2, port_vocab=l2p, V=V, ncols=V, eos=2, disabled=[0, 1, 2])
    return f, [llama3, llama2]


def bit_row(row, L):
    """A logits row in the port's bit space: bit t = column t, bit V = EOS column."""
    out = np.zeros(L["V"] + 1, np.uint16)
    out[: L["V"]] = row[: L["V"]]
    out[L["V"]] = row[L["eos"]]
    return out


def to_col(t, L):
    return L["eos"] if t == L["V"] else t


@pytest.fixture(scope="module", params=["llama3", "llama2"])
def setup(request):
    f, ls = layouts()
    L = [x for x in ls if x["name"] == request.param][0]
    eng = pk.DeviceEngine(pk.Automaton.load(f), L["engine_vocab"], context_depth=8, num_columns=L["ncols"],
                          eos_column=L["eos"], disabled=L["disabled"])
    port = Port(f, L["port_vocab"])
    return L, eng, port


@pytest.mark.parametrize("K,B", [(8, 24), (2, 64)])
def test_masked_logits_follow_the_layout(setup, K, B):
    """Fused mask + -inf: regular columns by their bit, the EOS column by bit
    V, every other special column -inf; the bitmask keeps the reference
    layout and equals the port's.  K = 2 makes EOS context-dependent in most
    contexts (the EOS column's segment is then heavy: its item walks EOS on
    the stack while the overlapped accept waits for it)."""
    L, eng8, port = setup
    eng = eng8 if K == 8 else pk.DeviceEngine(pk.Automaton.load(json_flat()), L["engine_vocab"], context_depth=K,
                                               num_columns=L["ncols"], eos_column=L["eos"], disabled=L["disabled"])
    batch = eng.batch(B)
    g = torch.Generator(device=DEV).manual_seed(3)
    toks = torch.zeros(B, dtype=torch.int32, device=DEV)
    cfgs = [port.initial() for _ in range(B)]
    bm = torch.zeros((B, eng.W), dtype=torch.int32, device=DEV)
    counts = torch.zeros((B, 2 * batch.nseg), dtype=torch.int32, device=DEV)
    seen_eos = 0
    for s in range(14):
        lg = torch.randn((B, L["ncols"]), generator=g, device=DEV).to(torch.bfloat16)
        before = lg.float().cpu().numpy()
        batch.decode_step_stream_split(9, bitmask=bm, logits=lg, seg_counts=counts, tokens_out=toks)
        batch.check()
        got = bm.cpu().numpy().view(np.uint32)
        after = lg.float().cpu().numpy()
        tk = toks.cpu().numpy()
        for b in range(B):
            want = port.mask(cfgs[b])
            assert np.array_equal(got[b], want), (b, s)
            bits = np.unpackbits(want.view(np.uint8), bitorder="little")[: L["V"] + 1].astype(bool)
            allowed = np.zeros(L["ncols"], bool)
            allowed[: L["V"]] = bits[: L["V"]]
            allowed[L["eos"]] = bits[L["V"]]
            seen_eos += int(bits[L["V"]])
            assert np.array_equal(np.isneginf(after[b]), ~allowed | np.isneginf(before[b])), (b, s)
            assert np.array_equal(after[b][allowed], before[b][allowed])
            t = port.stream_pick(want, eng.structural, Port.stream_draw(9, b, s))
            assert tk[b] == (to_col(t, L) if t >= 0 else -1), (b, s)
            if t >= 0:
                port.accept_token(cfgs[b], t)
            if t < 0 or cfgs[b].status != 0:
                port.free(cfgs[b])
                cfgs[b] = port.initial()
            assert batch.get(b).stack == port.get(cfgs[b])[2]
    assert seen_eos > 0


def test_greedy_and_sampler_in_model_columns(setup):
    """Greedy argmax and the temperature/top-k/top-p sampler read the EOS
    logit from the EOS column, never pick a special, and return column ids;
    the port picks the same over the row mapped to bit space."""
    L, eng, port = setup
    B = 16
    for mode in ("greedy", "sample"):
        batch = eng.batch(B)
        cfgs = [port.initial() for _ in range(B)]
        toks = torch.zeros(B, dtype=torch.int32, device=DEV)
        bm = torch.zeros((B, eng.W), dtype=torch.int32, device=DEV)
        g = torch.Generator(device=DEV).manual_seed(11)
        for s in range(12):
            lg = torch.randn((B, L["ncols"]), generator=g, device=DEV)
            lg[:, L["V"]:] += 3.0  # specials look attractive: they must still never win
            lg = lg.to(torch.bfloat16)
            if mode == "greedy":
                batch.decode_step_greedy(lg, tokens_out=toks, bitmask=bm)
            else:
                batch.decode_step_sample(lg, temperature=0.9, top_k=40, top_p=0.95, seed=5, tokens_out=toks,
                                         bitmask=bm)
            batch.check()
            rows = lg.view(torch.int16).cpu().numpy().view(np.uint16)
            tk = toks.cpu().numpy()
            for b in range(B):
                m = port.mask(cfgs[b])
                r = bit_row(rows[b], L)
                if mode == "greedy":
                    t = port.greedy_pick(m, r)
                else:
                    t = port.sample_pick(m, r, 0.9, 40, 0.95, Port.stream_draw(5, b, s))
                assert tk[b] == (to_col(t, L) if t >= 0 else -1), (mode, b, s)
                if t >= 0:
                    port.accept_token(cfgs[b], t)
                if t < 0 or cfgs[b].status != 0:
                    port.free(cfgs[b])
                    cfgs[b] = port.initial()
                assert batch.get(b).stack == port.get(cfgs[b])[2]


def test_accept_takes_model_columns(setup):
    """gm_accept_tokens in column ids: the EOS column steps the end marker;
    a special column, a disabled id or an id past the row kills the
    sequence."""
    L, eng, port = setup
    batch = eng.batch(4)
    st = torch.zeros(4, dtype=torch.int32, device=DEV)
    bad_special = L["V"] if L["ncols"] > L["V"] else 0  # llama3: <|begin_of_text|>; llama2: <unk> (disabled)
    batch.accept(torch.tensor([bad_special, L["ncols"] + 5, 1 if L["disabled"] else L["V"] + 7, -1],
                              dtype=torch.int32, device=DEV), st)
    batch.check()
    assert st.cpu().tolist() == [pk.DEAD, pk.DEAD, pk.DEAD, pk.ALIVE]
    # '[' ']' then EOS (column) accepts the document
    lb, rb = L["engine_vocab"].index(b"["), L["engine_vocab"].index(b"]")
    b2 = eng.batch(1)
    s1 = torch.zeros(1, dtype=torch.int32, device=DEV)
    for t in (lb, rb, L["eos"]):
        b2.accept(torch.tensor([t], dtype=torch.int32, device=DEV), s1)
    b2.check()
    assert int(s1.item()) == pk.ACCEPTED

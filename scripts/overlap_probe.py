"""Step time of the two-kernel step with and without an event between the
kernels (PDL overlap of the accept with the fill's last wave)."""
import sys, os, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench, paper_2506_03887_b200 as pk
B = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
grammar = sys.argv[2] if len(sys.argv) > 2 else "json"
K = int(sys.argv[3]) if len(sys.argv) > 3 else 16
flat = bench.automaton_bytes(grammar)
vocab = pk.synth_vocab(128255)
eng = pk.DeviceEngine(pk.Automaton.load(flat), vocab, context_depth=K, context_slots=65536)
eng.prewarm(1024, 10000, seed=0xC0FFEE)
dev = torch.device("cuda:0")
batch = eng.batch(B)
W, V1 = eng.W, eng.V + 1
bm = torch.zeros((B, W), dtype=torch.int32, device=dev)
cn = torch.zeros((B, batch.nseg * 2), dtype=torch.int32, device=dev)
tk = torch.zeros(B, dtype=torch.int32, device=dev)
R = 3
lg = [torch.randn((B, V1), dtype=torch.bfloat16, device=dev) for _ in range(R)]
s = torch.cuda.current_stream()
for mid in (True, False, True, False):
    for i in range(30):
        batch.fill(bm, lg[i % R], cn); batch.sample_stream_and_accept(bm, cn, 1, tk)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    mids = [torch.cuda.Event(enable_timing=True) for _ in range(200)]
    e0.record(s)
    for i in range(200):
        batch.fill(bm, lg[i % R], cn)
        if mid:
            mids[i].record(s)
        batch.sample_stream_and_accept(bm, cn, 1, tk)
    e1.record(s)
    torch.cuda.synchronize()
    batch.check()
    print(f"B={B} {grammar} K={K} mid_event={mid}: step {e0.elapsed_time(e1) / 200 * 1e3:.1f} us")

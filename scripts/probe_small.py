"""GPU probe: latency of small parses (1 MB cfg1): eager parse_into, and a CUDA-graph replay of it."""
import sys, time
sys.path.insert(0, ".")
import torch
import datagen
import paper_1905_13415_b200 as parpa
name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
n = int(float(sys.argv[2])) if len(sys.argv) > 2 else 1_000_000
w = datagen.WORKLOADS[name]
data, g = datagen.generate(name, n)
d = torch.from_numpy(data.copy()).cuda()
dfa = parpa.Dfa.dialect(w.dialect)
schema = parpa.Schema(list(w.types))
cap = g.records + 2
cols = parpa.alloc_columns(schema, cap)
st = parpa.new_stats_tensor()
s = torch.cuda.current_stream()
for _ in range(5):
    parpa.parse_into(dfa, schema, d, cols, cap, st, stream=s)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
N = 200
t0 = time.perf_counter(); e0.record()
for _ in range(N):
    parpa.parse_into(dfa, schema, d, cols, cap, st, stream=s)
e1.record(); torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"eager: {e0.elapsed_time(e1) / N * 1e3:.1f} us/parse device, {(t1 - t0) / N * 1e6:.1f} us/parse wall, "
      f"{g.nbytes / (e0.elapsed_time(e1) / N * 1e-3) / 1e9:.1f} GB/s")
assert parpa.stats_from_tensor(st)["records"] == g.records
try:
    gs = torch.cuda.Stream()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.stream(gs):
        parpa.parse_into(dfa, schema, d, cols, cap, st, stream=gs)
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=gs):
            parpa.parse_into(dfa, schema, d, cols, cap, st, stream=gs)
    torch.cuda.synchronize()
    st.zero_()
    graph.replay(); torch.cuda.synchronize()
    assert parpa.stats_from_tensor(st)["records"] == g.records, parpa.stats_from_tensor(st)
    t0 = time.perf_counter(); e0.record()
    for _ in range(N):
        graph.replay()
    e1.record(); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"graph: {e0.elapsed_time(e1) / N * 1e3:.1f} us/parse device, {(t1 - t0) / N * 1e6:.1f} us/parse wall, "
          f"{g.nbytes / (e0.elapsed_time(e1) / N * 1e-3) / 1e9:.1f} GB/s")
except Exception as ex:
    print("graph capture failed:", repr(ex)[:300])

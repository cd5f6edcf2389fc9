"""GPU probe: device time of the τ-only (summarize) and τ+count (count) kernels."""
import sys
sys.path.insert(0, ".")
import torch
import datagen
import paper_1905_13415_b200 as parpa
name, n = sys.argv[1], int(float(sys.argv[2]))
w = datagen.WORKLOADS[name]
data, g = datagen.generate(name, n)
d = torch.from_numpy(data.copy()).cuda()
dfa = parpa.Dfa.dialect(w.dialect)
for fn, lab in ((lambda: parpa.summarize(dfa, d), "summarize"), (lambda: parpa.count(dfa, d, 0, 0), "count")):
    for rep in range(3):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); s.record(); fn(); e.record(); torch.cuda.synchronize()
    print(f"{name} {lab}: {s.elapsed_time(e):.3f} ms -> {n / s.elapsed_time(e) / 1e6:.0f} GB/s")

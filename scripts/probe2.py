"""GPU probe: per-kernel device times (CUDA events) for the fused and two-phase paths."""
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
schema = parpa.Schema(list(w.types))
cols = parpa.alloc_columns(schema, g.records + 1)
st = parpa.new_stats_tensor()
for rep in range(3):
    parpa.set_profiling(True)
    parpa.parse_into(dfa, schema, d, cols, g.records + 1, st)
    torch.cuda.synchronize()
    fused = parpa.last_kernel_times()
    parpa.set_profiling(True)
    r = parpa.parse(dfa, schema, d)
    torch.cuda.synchronize()
    plan = parpa.last_kernel_times()
    parpa.set_profiling(False)
s = parpa.stats_from_tensor(st)
assert s["status"] == 0 and s["records"] == g.records and r.records == g.records
fmt = lambda kt: " ".join(f"{k}={v:.3f}ms" for k, v in kt)
gbs = lambda kt, key: n / (sum(v for k, v in kt if k.startswith(key)) * 1e-3) / 1e9
print(f"{name} {n/1e9:.2f}GB fused: {fmt(fused)}  -> scan {gbs(fused,'k_scan'):.0f} GB/s")
print(f"{name} {n/1e9:.2f}GB plan:  {fmt(plan)}  -> scan {gbs(plan,'k_scan'):.0f} GB/s, emit {gbs(plan,'k_emit'):.0f} GB/s")

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
fmt = lambda kt: " ".join(f"{k}={v:.3f}" for k, v in kt)
tot = lambda kt: sum(v for k, v in kt)
print(f"{name} {n/1e9:.2f}GB into: {tot(fused):.3f} ms -> {n / tot(fused) / 1e6:.0f} GB/s   [{fmt(fused)}]")
print(f"{name} {n/1e9:.2f}GB plan: {tot(plan):.3f} ms -> {n / tot(plan) / 1e6:.0f} GB/s   [{fmt(plan)}]")

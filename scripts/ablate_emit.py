"""GPU probe: k_emit time on taxi-shaped input under schema variants (where does the emit time go?).
usage: python scripts/ablate_emit.py [bytes]"""
import sys

sys.path.insert(0, ".")
import torch

import datagen
import paper_1905_13415_b200 as parpa

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 2e9
w = datagen.WORKLOADS["taxi"]
data, g = datagen.generate("taxi", n)
d = torch.from_numpy(data.copy()).cuda()
dfa = parpa.Dfa.dialect(w.dialect)
S = datagen.SPAN
variants = {
    "full": list(w.types),
    "all_span": [S] * w.C,
    "ints_only": [t if t == datagen.INT64 else S for t in w.types],
    "floats_only": [t if t == datagen.FLOAT64 else S for t in w.types],
    "one_col": list(w.types),          # all columns counted, only column 0 written (NULL pointers)
}
for name, types in variants.items():
    schema = parpa.Schema(types)
    cols = parpa.alloc_columns(schema, g.records + 1)
    if name == "one_col":
        cols = [cols[0]] + [parpa.Column(None, None)] * (w.C - 1)
    st = parpa.new_stats_tensor()
    best = None
    for rep in range(4):
        parpa.set_profiling(True)
        parpa.parse_into(dfa, schema, d, cols, g.records + 1, st)
        torch.cuda.synchronize()
        kt = dict(parpa.last_kernel_times())
        parpa.set_profiling(False)
        if rep and (best is None or kt["k_emit"] < best):
            best = kt["k_emit"]
    print(f"{name:12s} k_emit {best:.3f} ms  ({n / best / 1e6:.0f} GB/s of input)", flush=True)

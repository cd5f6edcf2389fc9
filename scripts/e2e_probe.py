"""End-to-end probe: parpa_parse_host wall time for taxi at several partition sizes."""
import os
import sys
import time

sys.path.insert(0, ".")
import torch

import bench
import datagen
import paper_1905_13415_b200 as parpa

cfg = sys.argv[1] if len(sys.argv) > 1 else "taxi"
w = datagen.WORKLOADS[cfg]
data_host, _, _, _, g = bench.gen_range(cfg, 0, 1)
dfa = parpa.Dfa.dialect(w.dialect)
schema = parpa.Schema(list(w.types))
cap = g.records
host_cols = []
for t in w.types:
    off = torch.empty(cap, dtype=torch.int64, pin_memory=True)
    ln = torch.empty(cap, dtype=torch.int32, pin_memory=True)
    if t == datagen.SPAN:
        host_cols.append(parpa.Column(off, ln))
    else:
        host_cols.append(parpa.Column(off, ln, torch.empty(cap, dtype=torch.int64, pin_memory=True),
                                      torch.empty(cap, dtype=torch.uint8, pin_memory=True)))
for P in [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["536870912"])]:
    os.environ["PARPA_STREAM_PARTITION"] = str(P)
    ts = []
    for i in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = parpa.parse_host_into(dfa, schema, data_host, host_cols, cap)
        ts.append(time.perf_counter() - t0)
        assert st["status"] == 0 and st["records"] == cap, st
    print(f"{cfg} partition {P >> 20} MB: " + " ".join(f"{t * 1e3:.0f}" for t in ts) + f" ms -> {data_host.numel() / min(ts[1:]) / 1e9:.2f} GB/s", flush=True)

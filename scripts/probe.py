"""Quick GPU probe: parse a generated workload of a given size through both paths, print timings."""
import sys
import time

sys.path.insert(0, ".")
import torch

import datagen
import paper_1905_13415_b200 as parpa

name, n, path = sys.argv[1], int(float(sys.argv[2])), sys.argv[3]
w = datagen.WORKLOADS[name]
data, g = datagen.generate(name, n)
d = torch.from_numpy(data.copy()).cuda()
dfa = parpa.Dfa.dialect(w.dialect)
schema = parpa.Schema(list(w.types))
torch.cuda.synchronize()
t0 = time.time()
if path == "plan":
    r = parpa.parse(dfa, schema, d)
    st = r.stats
elif path == "tau":
    tau = parpa.summarize(dfa, d)
    st = {"tau": tau, "records": g.records, "status": 0}
elif path == "count":
    c, tau = parpa.count(dfa, d, 0, 0)
    st = {"records": c.records, "status": 0, "tau": tau}
else:
    cols = parpa.alloc_columns(schema, g.records + 1)
    s = parpa.new_stats_tensor()
    parpa.parse_into(dfa, schema, d, cols, g.records + 1, s)
    st = parpa.stats_from_tensor(s)
torch.cuda.synchronize()
print(name, n, path, "ok" if st["status"] == 0 and st["records"] in (g.records,) else "MISMATCH", st["records"], g.records,
      f"{(time.time() - t0) * 1e3:.1f} ms", flush=True)

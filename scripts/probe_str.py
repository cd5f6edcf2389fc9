import sys; sys.path.insert(0, '.')
import torch, numpy as np, datagen, oracle, paper_1905_13415_b200 as parpa
name = sys.argv[1]; n = int(float(sys.argv[2])); cols = [int(c) for c in sys.argv[3].split(',')]
w = datagen.WORKLOADS[name]
data, g = datagen.generate(name, n)
d = torch.from_numpy(data.copy()).cuda()
dfa = parpa.Dfa.dialect(w.dialect)
res = parpa.parse(dfa, parpa.Schema(list(w.types)), d)
for c in cols:
    try:
        offs, buf = parpa.strings(dfa, d, res.columns[c], res.records)
        ro, rs = oracle.strings(w.dialect, data, w.C, c, list(w.types))
        print(c, np.array_equal(offs.cpu().numpy(), ro), bytes(buf.cpu().numpy()) == rs)
    except Exception as e:
        print(c, "ERR", e, parpa.last_error() if hasattr(parpa, "last_error") else "")
        raise

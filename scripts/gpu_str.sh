cd $GRAFT_REPO_ROOT
timeout 500 python -m pytest tests -m gpu -q -x --timeout 200 2>&1 | tail -2
cat > /tmp/strbench.py <<'PY'
import sys; sys.path.insert(0, '.')
import torch, datagen, paper_1905_13415_b200 as parpa
w = datagen.WORKLOADS['yelp']; data, g = datagen.generate('yelp', 4_823_000_000)
d = torch.from_numpy(data).cuda(); del data
dfa = parpa.Dfa.dialect('csv'); res = parpa.parse(dfa, parpa.Schema(list(w.types)), d)
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    offs, buf = parpa.strings(dfa, d, res.columns[7], res.records)
    e1.record(); torch.cuda.synchronize()
print(f"yelp text column: {res.records} rows, {buf.numel()/1e9:.2f} GB of strings in {e0.elapsed_time(e1):.2f} ms (size + copy, incl. the scan half twice)")
PY
timeout 300 python /tmp/strbench.py 2>&1 | tail -1

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
cat > /tmp/one.py <<'PY'
import sys; sys.path.insert(0,'.')
import torch, datagen, paper_1905_13415_b200 as parpa
name=sys.argv[1]
w=datagen.WORKLOADS[name]; data,g=datagen.generate(name, 1_000_000_000)
d=torch.from_numpy(data.copy()).cuda(); dfa=parpa.Dfa.dialect(w.dialect); sch=parpa.Schema(list(w.types))
for i in range(3): r=parpa.parse(dfa, sch, d)
torch.cuda.synchronize(); print(r.records)
PY
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_pass -s 4 -c 2 -o gpurun_out/prof_pass_$1 python /tmp/one.py $1 > gpurun_out/ncu_p.log 2>&1; echo ncu rc=$?

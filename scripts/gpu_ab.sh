cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in A B C; do
  if [ $v = A ]; then unset PARPA_LIB; else export PARPA_LIB=$PWD/abtest/lib$v.so; fi
  for w in yelp taxi clf; do echo -n "$v "; timeout 120 python scripts/probe2.py $w 2e9 2>&1 | grep -E "GB|Error" | tail -2 | tr '\n' ' '; echo; done
done
unset PARPA_LIB
cat > /tmp/one.py <<'PY'
import sys; sys.path.insert(0,'.')
import torch, datagen, paper_1905_13415_b200 as parpa
name=sys.argv[1]
w=datagen.WORKLOADS[name]; data,g=datagen.generate(name, 1_000_000_000)
d=torch.from_numpy(data.copy()).cuda(); dfa=parpa.Dfa.dialect(w.dialect); sch=parpa.Schema(list(w.types))
cols=parpa.alloc_columns(sch, g.records+1); st=parpa.new_stats_tensor()
for i in range(3): parpa.parse_into(dfa, sch, d, cols, g.records+1, st)
torch.cuda.synchronize(); print(parpa.stats_from_tensor(st))
PY
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_scan -s 2 -c 1 -o gpurun_out/prof_fused_yelp python /tmp/one.py yelp > gpurun_out/ncu_fy.log 2>&1; echo ncu rc=$?

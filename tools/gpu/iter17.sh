cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_spmm_groups.py -q -m gpu --timeout 900 2>&1 | tail -3
timeout 900 python tools/bench_offline.py > gpurun_out/offline.json 2>&1
python -c "
import json; o=json.load(open('gpurun_out/offline.json'))
for k in (8,32,400):
  print(k, {t: (round(o.get(f'spmm{t}_k{k}_ms',0),3), round(o.get(f'spmm{t}_k{k}_frac_hbm',0),3), round(o.get(f'spmm{t}_k{k}_frac_fp64',0),3)) for t in ('','_rgtc','_rgcc','_rgcc_direct')})
"

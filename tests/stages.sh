# tile-sort stage timings (tuning aid): NSB_TS_STAGE / NSB_TS_KB knobs
for cfg in "0 1" "0 23" "0 31" "2 1"; do set -- $cfg; NSB_TS_STAGE=$1 NSB_TS_KB=$2 timeout 120 python - <<'PY'
import os,sys,torch
sys.path.insert(0,'.')
import paper_2503_05934_b200 as ns
from paper_2503_05934_b200._lib import check
L=ns.lib(); n=1<<28
a=torch.empty(n,dtype=torch.int32,device='cuda'); check(L.ns_generate_i32(a.data_ptr(),n,0,42,0),'g')
w=a.clone(); cfg=ns.find_config('6To8')
for seg in (8192,16384):
  ts=[]
  for i in range(4):
    w.copy_(a); e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
    e0.record(); ns.segmented_sort(w, seg, cfg, ns.Algorithm.merge_sort); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
  print('stage', os.environ['NSB_TS_STAGE'], 'kb', os.environ['NSB_TS_KB'], 'seg', seg, 'ms', round(min(ts[1:]),4))
PY
done

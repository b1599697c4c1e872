o=gpurun_out/${1:-n3d}; mkdir -p $o
cat > $o/prof.py <<'PY'
import sys; sys.path.insert(0,'.')
import torch
from paper_2311_03906_b200 import Sampler, circuits as CI, run_initialization
init=run_initialization(CI.CONFIGS["cfg3"]["text"]()); s=Sampler(init)
dets,obs=CI.surface_code_detectors(15,15); s.set_detectors(dets+obs)
n=2000000; T=s.shot_tile; n=(n+T-1)//T*T
out=torch.empty(s.tiled_words(n),dtype=torch.int64,device="cuda"); dc=torch.zeros(len(dets)+1,dtype=torch.int64,device="cuda")
for i in range(2): s.sample_counted(n, 10+i, out=out, det_counts=dc, tiled=True)
torch.cuda.synchronize(); print("ok", s.plan_info())
PY
SP_AUTOTUNE=0 SP_GEN_WARPS=${GW:-10} SP_PAD_PRED=${PP:-0} ncu --set full --import-source on --clock-control none -k regex:k1_fused -s 1 -c 1 -o $o/k1 python $o/prof.py > $o/ncu.log 2>&1
python tools/ncu_summarize.py $o/k1.ncu-rep > $o/summary.txt 2>&1
python tools/ncu_regions.py $o/k1.ncu-rep > $o/regions.txt 2>&1

# One ncu --set full capture of the fused sampler the cfg3 bench runs (tiled records, detector counts):
#   tools/ncu_bench_kernel.sh OUTDIR SHOTS [k7|k1]
o=gpurun_out/${1:-nbk}; n=${2:-2000000}; k=${3:-k7}; mkdir -p $o
cat > $o/prof.py <<PY
import sys; sys.path.insert(0,'.')
import torch
from paper_2311_03906_b200 import Sampler, circuits as CI, run_initialization
init=run_initialization(CI.CONFIGS["cfg3"]["text"]()); s=Sampler(init)
dets,obs=CI.surface_code_detectors(15,15); s.set_detectors(dets+obs)
n=$n; T=s.shot_tile; n=(n+T-1)//T*T
out=torch.empty(s.tiled_words(n),dtype=torch.int64,device="cuda"); dc=torch.zeros(len(dets)+1,dtype=torch.int64,device="cuda")
for i in range(2): s.sample_counted(n, 10+i, out=out, det_counts=dc, tiled=True)
torch.cuda.synchronize(); print("ok", n, s.plan_info())
PY
if [ $k = k7 ]; then export SP_QUEUED=1; re=k7_queued; else export SP_QUEUED=0 SP_GEN_WARPS=${GW:-10}; re=k1_fused; fi
SP_AUTOTUNE=0 ncu --set full --import-source on --clock-control none -k regex:$re -s 1 -c 1 -o $o/$k python $o/prof.py > $o/ncu_$k.log 2>&1
python tools/ncu_summarize.py $o/$k.ncu-rep > $o/summary_$k.txt 2>&1
python tools/ncu_regions.py $o/$k.ncu-rep > $o/regions_$k.txt 2>&1
ncu -i $o/$k.ncu-rep --page details --section SpeedOfLight --print-details all > $o/sol_$k.txt 2>&1
tail -n 2 $o/ncu_$k.log

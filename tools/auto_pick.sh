# What the launch autotune picks (K1 or K7) for each workload's launch kind and the resulting kernel time.
# Three fresh processes per workload.
o=gpurun_out/${1:-ap}; mkdir -p $o
for rep in 1 2 3; do
for cfg in "cfg3 --shots 10000000 --tiled --dets" "cfg3 --shots 10000000 --tiled" "cfg2 --shots 10002432 --dets" "cfg2 --shots 10002432" "cfg4 --shots 1000000 --tiled" "cfg1 --shots 1000000"; do
timeout 200 python tools/time_kernel.py --config $cfg --reps 5 2>>$o/err.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['plan']
print('rep $rep', '$cfg', 'ms', round(d['ms_median'],4), d['kernel'], 'plan sampler code', p['fused_ok'])" >> $o/t.txt 2>&1
done; done
cat $o/t.txt

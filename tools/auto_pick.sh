# What the launch autotune picks (K1 or K7) and the resulting kernel time, per workload.
o=gpurun_out/${1:-ap}; mkdir -p $o
for cfg in "cfg3 --shots 10000000 --tiled --dets" "cfg3 --shots 10000000 --tiled" "cfg2 --shots 10002432 --dets" "cfg2 --shots 10002432" "cfg4 --shots 1000000 --tiled" "cfg1 --shots 1000000"; do
timeout 200 python tools/time_kernel.py --config $cfg --reps 5 2>>$o/err.txt | python -c "
import json,sys; d=json.loads(sys.stdin.read()); p=d['plan']
print('$cfg', 'ms', round(d['ms_median'],4), 'sampler', p['fused_ok'], 'warps', p['gen_warps'], 'threads', p['cta_threads'])" >> $o/t.txt 2>&1
done
cat $o/t.txt

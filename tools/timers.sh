o=gpurun_out/${1:-tm}; mkdir -p $o
for x in "" "--dets"; do for bk in 0 1; do
SP_BULK=$bk SP_PHASE_TIMERS=1 SP_AUTOTUNE=0 SP_GEN_WARPS=11 python tools/time_kernel.py --config cfg3 --shots 10000000 --tiled $x --reps 3 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); t=d['timers']; g=d['plan']['gen_warps']; dr=16-g
print('x=$x bulk=$bk', round(d['ms_median'],3), 'gen wait/work per warp %.2f/%.2f G' % (t[0]/g/1e9, t[1]/g/1e9), 'drain wait/work per warp %.2f/%.2f G' % (t[2]/dr/1e9, t[3]/dr/1e9))" >> $o/t.txt 2>&1
done; done
cat $o/t.txt

o=gpurun_out/${1:-tm}; mkdir -p $o
for x in "" "--dets"; do for gw in 10 11 12 13; do
SP_PHASE_TIMERS=1 SP_AUTOTUNE=0 SP_GEN_WARPS=$gw python tools/time_kernel.py --config cfg3 --shots 10000000 --tiled $x --reps 3 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); t=d['timers']; g=d['plan']['gen_warps']; dr=16-g
tot=(t[0]+t[1])/g
print('x=$x gw=$gw', round(d['ms_median'],3), 'gen wait/work %.0f%%/%.0f%%' % (100*t[0]/g/tot, 100*t[1]/g/tot), 'drain wait/work %.0f%%/%.0f%%' % (100*t[2]/dr/tot, 100*t[3]/dr/tot))" >> $o/t.txt 2>&1
done; done
cat $o/t.txt

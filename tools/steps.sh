# Walk steps and firings per shot (SP_PHASE_TIMERS counters [4], [5]) at cfg2/cfg3/cfg4.
o=gpurun_out/${1:-steps}; mkdir -p $o
for cfg in "cfg3 --shots 10000000 --tiled" "cfg2 --shots 10002432" "cfg4 --shots 1000000 --tiled"; do
SP_PHASE_TIMERS=1 python tools/time_kernel.py --config $cfg --reps 1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); t=d['timers']; n=d.get('shots') or 1
print('$cfg', 'ms', round(d['ms_median'],3), 'steps', t[4], 'firings', t[5], 'firings/step %.1f' % (t[5]/max(t[4],1)), 'plan', d['plan'])" >> $o/t.txt 2>&1
done
cat $o/t.txt

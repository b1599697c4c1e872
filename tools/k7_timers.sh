# K7 per-tile phase cycles (SP_PHASE_TIMERS): apply waiting for an empty buffer / whole tile, drain waiting
# for full / working, rebuild phase, TMA read wait. Per tile per warp (or per elected thread).
o=gpurun_out/${1:-k7t}; mkdir -p $o
for m in ${2:-0 6}; do
SP_QUEUED=1 SP_DEBUG_MODE=$m SP_PHASE_TIMERS=1 timeout 120 python tools/time_kernel.py --config cfg3 --shots 10000000 --tiled --reps 1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); t=d['timers']; runs=4; tiles=d['shots']/128*runs
napp=8; ndr=16
print('mode=$m ms', round(d['ms_median'],3), 'per tile: apply empty-wait %.0f, apply tile %.0f | drain full-wait %.0f work %.0f | rebuild %.0f, tma read wait %.0f  (clk)' % (t[0]/napp/tiles, t[1]/napp/tiles, t[2]/ndr/tiles, t[3]/ndr/tiles, t[6]/tiles, t[7]/tiles), 'per-CTA tile period %.0f clk' % (d['ms_median']*1e-3*1.965e9/(d['shots']/128/148)))" >> $o/t.txt 2>&1
done
cat $o/t.txt

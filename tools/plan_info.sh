o=gpurun_out/${1:-pi}; mkdir -p $o
for e in "SP_MECH=1" "SP_MECH=0"; do
env $e SP_PHASE_TIMERS=1 python tools/time_kernel.py --config cfg3 --shots 10000000 --tiled --reps 3 > $o/cfg3_$e.json 2>&1
env $e SP_PHASE_TIMERS=1 python tools/time_kernel.py --config cfg2 --shots 10002432 --reps 3 > $o/cfg2_$e.json 2>&1
done
cat $o/*.json

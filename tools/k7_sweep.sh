# K7 shape sweep at cfg3 (tiled, detector counts): walkers x apply warps x ring depth x threads.
o=gpurun_out/${1:-k7s}; mkdir -p $o
run() { env "$@" timeout 120 python tools/k7_check.py --config cfg3 --shots 10000000 --tiled --dets --no-check --reps 3 2>>$o/err.txt | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(' '.join(f'{k}={v}' for k,v in d['env'].items()), 'k1', round(d['k1_ms'],3), 'k7', round(d['k7_ms'],3))" >> $o/t.txt; }
for cfgs in "8 8 8" "8 16 8" "10 10 8" "12 12 8" "12 12 4" "14 14 4" "16 8 4" "10 10 4" "8 16 16" ; do
set -- $cfgs
run SP_Q_THREADS=1024 SP_Q_WALK=$1 SP_Q_APPLY=$2 SP_Q_DEPTH=$3
done
run SP_Q_THREADS=768 SP_Q_WALK=8 SP_Q_APPLY=8 SP_Q_DEPTH=8
run SP_Q_THREADS=768 SP_Q_WALK=10 SP_Q_APPLY=10 SP_Q_DEPTH=4
cat $o/t.txt

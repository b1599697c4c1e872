# K7 shape sweep at cfg3 (tiled, detector counts): "walkers apply depth" triples (1024 threads; the rest drain).
# usage: tools/k7_sweep.sh OUTDIR "8 8 4" "6 6 8" ...   (other SP_* switches from the environment)
o=gpurun_out/${1:-k7s}; shift; mkdir -p $o
for shape in "$@"; do
set -- $shape
env SP_Q_THREADS=1024 SP_Q_WALK=$1 SP_Q_APPLY=$2 SP_Q_DEPTH=$3 timeout 120 python tools/k7_check.py --config cfg3 --shots 10000000 --tiled --dets --no-check --reps 3 2>>$o/err.txt | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print(' '.join(f'{k}={v}' for k,v in d['env'].items() if k!='SP_QUEUED'), 'k1', round(d['k1_ms'],3), 'k7', round(d['k7_ms'],3))" >> $o/t.txt
done
cat $o/t.txt

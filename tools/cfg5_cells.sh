# cfg5: sp_sample (the planner's pick: 1 K1, 2 K5, 0 draw + explicit product) over the 9 (density, p) cells.
o=gpurun_out/${1:-c5}; mkdir -p $o
for d in 0.001 0.01 0.5; do for p in 1e-4 1e-3 1e-2; do
  python tools/k5_time.py $d $p 2>&1 | tail -1
done; done > $o/cells.jsonl
cat $o/cells.jsonl

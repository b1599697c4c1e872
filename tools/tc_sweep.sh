# K6 vs K2 (Four-Russians) over shapes: which dense product AUTO should pick.
o=gpurun_out/tcs; mkdir -p $o
for shape in "1000 10000" "1000 100000" "10000 10000" "3000 30000" "10000 100000" "100 100000" "10000 1000"; do
  for n in 65536 1048576; do
    python tools/tc_time.py $n 0.5 $shape 2>&1 | tr '\n' ' '; echo
  done
done > $o/sweep.txt

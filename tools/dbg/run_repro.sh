#!/bin/bash
for p in 1e-09 1e-06 0.0001; do
  echo "== p=$p"; timeout 120 python tools/dbg/repro_tiny.py $p 2>&1 | tail -30
  echo "== p=$p SP_AUTOTUNE=0"; SP_AUTOTUNE=0 timeout 120 python tools/dbg/repro_tiny.py $p 2>&1 | tail -8
done

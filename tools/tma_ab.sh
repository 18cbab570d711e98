#!/bin/bash
# A/B of the TMA tensor-store path (RS_TMA=1), per-lane bulk copies (RS_TMA=2) and the
# shared-tile STG path (default), same build
for cfg in "x256** uint64 30 --seed 12345" "x256** u01 30" "pcg64 uint64 30" "ranlux++ uint64 28" "x256** u01f 30" "xoro++ uint64 30"; do
  printf "tma    "; RS_TMA=1 python tools/profile_fill.py $cfg --reps 4 2>&1 | tail -1
  printf "bulk   "; RS_TMA=2 python tools/profile_fill.py $cfg --reps 4 2>&1 | tail -1
  printf "stg    "; python tools/profile_fill.py $cfg --reps 4 2>&1 | tail -1
done
for m in 6 1000003; do
  printf "tma    c5b m=$m "; RS_TMA=1 python tools/streams_fill.py $m --time 2>&1 | tail -1
  printf "stg    c5b m=$m "; python tools/streams_fill.py $m --time 2>&1 | tail -1
done

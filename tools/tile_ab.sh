#!/bin/bash
# A/B of the warp-tile parse (RS_TILE=1, opt-in) against the two-pass path, same build
for cfg in "pcg64 norm 28" "pcg64 exp 26" "philox norm 28" "pcg64 uint64 28 b=6" "pcg64 uint64 28 b=9223372036854775809" "philox exp 26" "pcg64 lognormal 26"; do
  printf "tile   "; RS_TILE=1 python tools/profile_fill.py $cfg --reps 4 2>&1 | tail -1
  printf "2pass  "; python tools/profile_fill.py $cfg --reps 4 2>&1 | tail -1
done

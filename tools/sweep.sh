#!/bin/bash
# one-line timings of a set of fills (tools/profile_fill.py, CUDA events, best of 3)
while read -r line; do
  [ -z "$line" ] && continue
  python tools/profile_fill.py $line --reps 3 2>&1 | tail -1
done <<'LIST'
x256++simd uint64 30
x256++simd u01 30
x256++simd u01f 30
x256++simd norm 28
x256**simd norm 28
sfc64simd uint64 24
x128+ uint64 30
xoro++ u01 30
xoro++ norm 28
squares uint64 30
squares norm 28
chacha20 uint64 30
chacha20 norm 28
cwg128 uint64 20
pcg64 uint64 28 b=6
pcg64 uint64 28 b=9223372036854775809
x256** normf 28
pcg64 u01f 30
x256** lognormal 26
pcg64 chi2 26 nu=3
LIST

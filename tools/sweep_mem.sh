while read -r line; do [ -z "$line" ] && continue; python tools/profile_fill.py $line --reps 3 2>&1 | tail -1; done <<'LIST'
x256++simd norm 28
philox norm 28
ranlux++ norm 26
chacha20 norm 28
xoro++ norm 28
x256++simd gamma 26 alpha=2.5
philox exp 26
x256** norm 28
LIST

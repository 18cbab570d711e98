#!/bin/bash
# Per-config instruction counts for the issue roofline in bench.py: every kernel of each BASELINE
# parse / per-stream fill under `ncu --metrics` (one rep, same seeds as bench.py), summed per
# config by tools/issue_counts.py into profiles/r02_issue_counts.json.
#   bash tools/issue_counts.sh OUTDIR
out=${1:-gpurun_out/issue}
mkdir -p "$out"
M=smsp__inst_executed.sum,smsp__thread_inst_executed.sum,gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
run() { # label, command...
  local label=$1; shift
  ncu --metrics $M --clock-control none --csv --log-file "$out/$label.csv" "$@" > /dev/null 2>&1
}
run c1_x256ss_raw_u64_2p30 python tools/profile_fill.py 'x256**' uint64 30 --reps 1 --seed 12345
run c2_philox_u01_f64_2p30 python tools/profile_fill.py philox u01 30 --reps 1 --seed 7 --fm
run c2_philox_u01f_f32_2p30 python tools/profile_fill.py philox u01f 30 --reps 1 --seed 7 --fm
run c3_x256ss_norm_2p28 python tools/profile_fill.py 'x256**' norm 28 --reps 1 --seed 2024
run c3_pcg64_norm_2p28 python tools/profile_fill.py pcg64 norm 28 --reps 1 --seed 2024
run c4_pcg64_exp_2p26 python tools/profile_fill.py pcg64 exp 26 --reps 1 --seed 99
for k in 0.3 1 2.5 10; do
  run c4_pcg64_gamma_${k}_2p26 python tools/profile_fill.py pcg64 gamma 26 alpha=$k --reps 1 --seed 99
done
run c4_pcg64_beta_2_5_2p26 python tools/profile_fill.py pcg64 beta 26 a=2 b=5 --reps 1 --seed 99
run extra_ranlux_raw_2p30 python tools/profile_fill.py ranlux++ uint64 30 --reps 1 --seed 12345
for m in 6 1000003 9223372036854775809; do
  run c5b_sfc64_streams_lemire_${m}_2p28 python tools/streams_fill.py $m
done
run c5a_z_philox_norm_2p29 python tools/profile_fill.py philox norm 29 --reps 1 --seed 31
echo done

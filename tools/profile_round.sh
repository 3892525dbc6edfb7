#!/bin/bash
# Full evidence run on one B200 (used through gpurun):
#   the GPU test suite, bench lines for C2..C5 and the reference arm, the ncu
#   launch list of the headline bench command, one `ncu --set full` capture per
#   top kernel (query-from-structures step and suffix-sort step), and a
#   compute-sanitizer memcheck + racecheck of tools/sanitize_smoke.py.
# usage: bash tools/profile_round.sh <outdir>      (e.g. gpurun_out/r02)
set -u
out=${1:-gpurun_out/prof}
mkdir -p "$out"
python -m pytest tests -m gpu -q > "$out/pytest_gpu.log" 2>&1; tail -1 "$out/pytest_gpu.log"
python bench.py > "$out/bench_C3.json" 2> "$out/bench_C3.err" || exit 1
for c in C2 C4 C5; do
  python bench.py --config $c --no-cpu-baseline > "$out/bench_$c.json" 2> "$out/bench_$c.err"
done
python bench.py --impl reference > "$out/bench_ref.json" 2> "$out/bench_ref.err"
# launch list of the same command (per-launch times are cold-cache and serialised)
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file "$out/launches.csv" \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > "$out/ncu_launches.log" 2>&1
python tools/ncu_step.py --query-only > "$out/step_plain.log" 2>&1 || exit 1
for spec in "k_query_fused 1 query" "k_raw_sa_emit 1 raw_sa_emit" "k_bucket_apply 1 bucket_apply"; do
  set -- $spec
  ncu --set full --clock-control none --import-source on -k regex:$1 --launch-skip $2 -c 1 \
      -o "$out/$3" python tools/ncu_step.py --query-only > "$out/$3.log" 2>&1
done
for spec in "k_onesweep 2 onesweep" "k_update 1 update" "k_small_groups 0 small_groups"; do
  set -- $spec
  ncu --set full --clock-control none --import-source on -k regex:$1 --launch-skip $2 -c 1 \
      -o "$out/$3" python tools/ncu_step.py > "$out/$3.log" 2>&1
done
timeout 1800 compute-sanitizer --tool memcheck --leak-check full python tools/sanitize_smoke.py \
    > "$out/sanitize_memcheck.log" 2>&1; echo "memcheck rc=$?" >> "$out/sanitize_memcheck.log"
timeout 1800 compute-sanitizer --tool racecheck python tools/sanitize_smoke.py \
    > "$out/sanitize_racecheck.log" 2>&1; echo "racecheck rc=$?" >> "$out/sanitize_racecheck.log"
ls "$out"

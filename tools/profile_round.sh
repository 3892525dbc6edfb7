#!/bin/bash
# Full evidence run on one B200 (used through gpurun):
#   bench lines for C2..C5, the ncu launch list of the headline bench command,
#   and one `ncu --set full` capture per top kernel of one C3 step.
# usage: bash tools/profile_round.sh <outdir>      (e.g. gpurun_out/r01)
set -u
out=${1:-gpurun_out/prof}
mkdir -p "$out"
python -m pytest tests -m gpu -x -q > "$out/pytest_gpu.log" 2>&1; tail -1 "$out/pytest_gpu.log"
python bench.py > "$out/bench_C3.json" 2> "$out/bench_C3.err" || exit 1
for c in C2 C4 C5; do
  python bench.py --config $c --no-cpu-baseline > "$out/bench_$c.json" 2> "$out/bench_$c.err"
done
python bench.py --impl reference > "$out/bench_ref.json" 2> "$out/bench_ref.err"
# launch list of the same command (per-launch times are cold-cache and serialised)
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file "$out/launches.csv" \
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline > "$out/ncu_launches.log" 2>&1
python tools/ncu_step.py > "$out/step_plain.log" 2>&1 || exit 1
for spec in "k_onesweep 2 onesweep" "k_query_fused 0 query" "k_update 1 update" "k_bucket_apply 0 bucket_apply" \
            "k_small_groups 0 small_groups" "k_onesweep 0 onesweep_text"; do
  set -- $spec
  ncu --set full --clock-control none --import-source on -k regex:$1 --launch-skip $2 -c 1 \
      -o "$out/$3" python tools/ncu_step.py > "$out/$3.log" 2>&1
done
ls "$out"

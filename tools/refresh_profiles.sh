#!/bin/bash
# Copy the evidence of one tools/profile_round.sh run into profiles/<round>/:
# bench lines, the raw launch list + its share table, per-kernel ncu summaries,
# raw metric pages and the DRAM traffic per launch that bench.py reports.
# usage: bash tools/refresh_profiles.sh gpurun_out/<run> profiles/r01
set -eu
src=$1
dst=${2:-profiles/r01}
mkdir -p "$dst"
for c in C2 C3 C4 C5 ref; do
  [ -s "$src/bench_$c.json" ] && cp "$src/bench_$c.json" "$dst/bench_$c.json"
done
gzip -c "$src/launches.csv" > "$dst/ncu_launches.csv.gz"
{
  echo 'Launch list: `ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline` (C3, 256 Mi i.i.d. DNA: structures built once, then query steps, then the end-to-end device steps and the e2e API calls). Per-launch times are cold-cache and serialised; compare shares, not absolutes.'
  echo
  python tools/launch_shares.py "$src/launches.csv"
} > "$dst/launch_shares.md"
reps=()
for r in query raw_sa_emit bucket_apply onesweep update small_groups onesweep_text; do
  [ -s "$src/$r.ncu-rep" ] || continue
  reps+=("$src/$r.ncu-rep")
  ncu -i "$src/$r.ncu-rep" --page raw --csv | gzip -c > "$dst/ncu_raw_k_$r.csv.gz"
done
python tools/ncu_summary.py "${reps[@]}" > "$dst/ncu_kernels.md"
args=()
for kv in "k_query_fused<true>=query" "k_raw_sa_emit=raw_sa_emit" "k_bucket_apply=bucket_apply" \
          "k_onesweep<u32>=onesweep" "k_update<false, unsigned>=update" "k_small_groups=small_groups"; do
  [ -s "$src/${kv#*=}.ncu-rep" ] && args+=("${kv%%=*}=$src/${kv#*=}.ncu-rep")
done
python tools/ncu_traffic.py "$dst/traffic.json" "${args[@]}"
for f in sanitize_memcheck.log sanitize_racecheck.log pytest_gpu.log; do
  [ -s "$src/$f" ] && cp "$src/$f" "$dst/$f"
done
# point each entry at the committed raw page (the .ncu-rep stays in gpurun_out)
python - "$dst/traffic.json" <<'PY'
import json, sys
d = json.load(open(sys.argv[1]))
for v in d.values():
    v["report"] = "ncu_raw_k_" + v["report"].replace(".ncu-rep", "") + ".csv.gz"
json.dump(d, open(sys.argv[1], "w"), indent=1)
PY
ls -la "$dst"

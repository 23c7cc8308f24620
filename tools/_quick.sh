# quick GPU iteration: tests (arg1 = pytest selection or "all"), bench C3 without CPU baseline, launch list
set -u
P=gpurun_out/q
mkdir -p $P
SEL=${1:-all}
if [ "$SEL" = "all" ]; then SEL="tests"; fi
if [ "$SEL" != "none" ]; then
timeout 900 python -m pytest $SEL -m gpu -q -x > $P/tests.log 2>&1; echo "tests rc=$?"; tail -3 $P/tests.log
fi
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline ${BENCH_ARGS:-} > $P/bench.json 2> $P/bench.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open("gpurun_out/q/bench.json").read().strip().splitlines()[-1])
print("ms", round(d["ms_per_step"],4), "breakdown", d["breakdown_ms"], "frac", round(d["roofline"]["frac"],3), "parity", d.get("parity"), "inc", {k: d["incremental"].get(k) for k in ("p50_ms","p99_ms","bit_exact_vs_full")} if d.get("incremental") else None, "e2e", d["e2e"]["ms_per_step"] if d.get("e2e") else None)
PY
if [ "${LAUNCHES:-1}" = "1" ]; then
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:fuse_|band_pass|refine_|gate_|tile_cull' --csv \
    --log-file $P/launches.csv python tools/profile_step.py --steps 2 > $P/ncu_l.log 2>&1; echo "launches rc=$?"
python tools/ncu_summary.py launches $P/launches.csv ""
fi

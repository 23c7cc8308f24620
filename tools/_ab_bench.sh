# A/B of library variants on the full bench step (graph, overlap); usage: bash tools/_ab_bench.sh v1 v2 ...
for rep in ${REPS:-1 2}; do
for v in "$@"; do
  if [ "$v" = cur ]; then unset DIVAS_LIB; else export DIVAS_LIB=/root/repo/_variants/$v.so; fi
  timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 ${BENCH_ARGS:-} 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['ms_per_step'],4), round(d['breakdown_ms']['refine'],4), round(d['breakdown_ms']['fuse'],4))"
done
done

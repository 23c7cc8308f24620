timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gt.txt 2>&1; tail -1 gpurun_out/gt.txt
for rep in 1 2 3; do for p in 0 1; do
  DIVAS_PDL=$p timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('pdl=$p', round(d['ms_per_step'],4), round(d['breakdown_ms']['refine'],4), round(d['breakdown_ms']['fuse'],4), d['probs_sha256'][:10], d['incremental']['p50_ms'])"
done; done

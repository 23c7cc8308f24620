set -u
P=gpurun_out/prof
mkdir -p $P
DIVAS_LIB=_variants/stats.so timeout 300 python tools/pair_stats.py --config C3 > $P/stats_C3.json 2>&1; echo "stats rc=$?"
timeout 300 python tools/profile_step.py --steps 2 > $P/step.log 2>&1; rc=$?; echo "step rc=$rc"
if [ $rc -eq 0 ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:fuse_|band_pass|refine_|gate_|tile_cull' --csv \
    --log-file $P/launches_C3.csv python tools/profile_step.py --steps 2 > $P/ncu_l.log 2>&1; echo "launches rc=$?"
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:fuse_pairs -s 1 -c 1 \
    -o $P/fuse_pairs python tools/profile_step.py --steps 2 > $P/ncu_f.log 2>&1; echo "full fuse_pairs rc=$?"
fi

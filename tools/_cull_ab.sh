for v in cur lb4 lb5; do
  if [ "$v" = cur ]; then unset DIVAS_LIB; else export DIVAS_LIB=/root/repo/_variants/$v.so; fi
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tile_cull --csv --log-file gpurun_out/tc_$v.csv python tools/profile_step.py --steps 3 >/dev/null 2>&1
  echo "$v $(python tools/launch_dram.py gpurun_out/tc_$v.csv)"
done
REPS="1 2 3" bash tools/_ab_bench.sh cur lb4 lb5

for v in cur g4b8 g2b8 g4b1; do
  if [ "$v" = cur ]; then unset DIVAS_LIB; else export DIVAS_LIB=/root/repo/_variants/$v.so; fi
  for c in C3 C5; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fuse_reduce --csv --log-file gpurun_out/rd_$v$c.csv python tools/profile_step.py --config $c --steps 2 >/dev/null 2>&1
  echo "$v $c $(python tools/launch_dram.py gpurun_out/rd_$v$c.csv)"
  done
done

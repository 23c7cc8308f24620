set -u
mkdir -p gpurun_out/q
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "regex:${KRE:-band_|refine_|gate_|fuse_|tile_cull}" --csv --log-file gpurun_out/q/l2.csv python tools/profile_step.py --steps 2 > gpurun_out/q/l2.log 2>&1; echo "rc=$?"

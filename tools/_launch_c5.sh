set -u
mkdir -p gpurun_out/q
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k "regex:band_|refine_|gate_|fuse_|tile_cull" --csv --log-file gpurun_out/q/c5.csv python tools/profile_step.py --config C5 --steps 1 > gpurun_out/q/c5.log 2>&1; echo "rc=$?"

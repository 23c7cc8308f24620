set -u
mkdir -p gpurun_out/q
timeout 300 python tools/profile_c4.py > gpurun_out/q/c4.log 2>&1; echo "c4 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k "regex:band_|refine_|gate_|fuse_|tile_cull|clear_view" --csv --log-file gpurun_out/q/c4.csv python tools/profile_c4.py > gpurun_out/q/c4n.log 2>&1; echo "ncu rc=$?"

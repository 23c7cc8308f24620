# Refresh the round's bench lines and ncu evidence (run on the GPU box via gpurun).
# Each ncu pass runs only after the same command exited 0 without ncu.
# usage: bash tools/refresh_profiles.sh [round-tag]   (default r02)
set -u
R=${1:-r02}
P=gpurun_out/prof_$R
mkdir -p $P
KRE='regex:fuse_|band_pass|refine_|gate_|tile_cull|band_init'
timeout 900 python bench.py > $P/bench_C3.json 2> $P/bench_C3.err; echo "bench C3 rc=$?"
timeout 900 python bench.py --impl reference > $P/bench_reference_C3.json 2> $P/bench_reference_C3.err; echo "ref rc=$?"
for c in C1 C2 C5; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline > $P/bench_$c.json 2> $P/bench_$c.err; echo "bench $c rc=$?"
done
DIVAS_FORCE_DIST=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu-baseline > $P/bench_dist1_C3_C5.json 2> $P/bench_dist1.err; echo "dist1 rc=$?"
timeout 300 python tools/profile_step.py --steps 2 > $P/step.log 2>&1; rc=$?; echo "step rc=$rc"
if [ $rc -eq 0 ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none -k "$KRE" --csv \
    --log-file $P/launches_C3.csv python tools/profile_step.py --steps 2 > $P/ncu_l.log 2>&1; echo "launches rc=$?"
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:fuse_pairs -s 1 -c 1 \
    -o $P/fuse_pairs python tools/profile_step.py --steps 2 > $P/ncu_f.log 2>&1; echo "full fuse_pairs rc=$?"
  timeout 900 ncu --set full --clock-control none -k 'regex:refine_minmax|band_pass|gate_tiles|gate_emit|fuse_reduce|tile_cull' \
    -c 6 -o $P/others python tools/profile_step.py --steps 1 > $P/ncu_o.log 2>&1; echo "full others rc=$?"
fi
timeout 300 python tools/profile_overlay.py > $P/overlay.log 2>&1; rc=$?; echo "overlay rc=$rc"
if [ $rc -eq 0 ]; then
  timeout 600 ncu --set full --clock-control none -k regex:overlay -c 1 -o $P/overlay python tools/profile_overlay.py > $P/ncu_ov.log 2>&1; echo "full overlay rc=$?"
fi

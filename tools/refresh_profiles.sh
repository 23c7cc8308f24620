# Refresh the round's bench lines and ncu evidence (run on the GPU box via gpurun).
# Each ncu pass runs only after the same command exited 0 without ncu.
set -u
P=gpurun_out/prof
mkdir -p $P
KRE='regex:fuse_|band_pass|refine_|gate_'
timeout 900 python bench.py > $P/bench_C3.json 2> $P/bench_C3.err; echo "bench C3 rc=$?"
timeout 600 python bench.py --impl reference > $P/bench_reference_C3.json 2> $P/bench_reference_C3.err; echo "ref rc=$?"
for c in C1 C2 C5; do
  timeout 900 python bench.py --config $c --steps 20 --warmup 3 > $P/bench_$c.json 2> $P/bench_$c.err; echo "bench $c rc=$?"
done
timeout 300 python tools/time_render.py --config C3 > $P/render_C3.json 2> $P/render_C3.err; echo "render C3 rc=$?"
timeout 300 python tools/time_render.py --config C5 --reps 3 > $P/render_C5.json 2> $P/render_C5.err; echo "render C5 rc=$?"
timeout 300 python tools/profile_step.py --steps 2 > $P/step.log 2>&1; rc=$?; echo "step rc=$rc"
if [ $rc -eq 0 ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KRE" --csv \
    --log-file $P/launches_C3.csv python tools/profile_step.py --steps 2 > $P/ncu_l.log 2>&1; echo "launches rc=$?"
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k "$KRE" --csv \
    --log-file $P/traffic_C3.csv python tools/profile_step.py --steps 2 > $P/ncu_t.log 2>&1; echo "traffic rc=$?"
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:fuse_pairs -s 1 -c 1 \
    -o $P/fuse_pairs python tools/profile_step.py --steps 2 > $P/ncu_f.log 2>&1; echo "full fuse_pairs rc=$?"
  timeout 900 ncu --set full --clock-control none -k 'regex:refine_minmax|band_pass|gate_tiles|gate_emit|fuse_reduce' \
    -c 5 -o $P/others python tools/profile_step.py --steps 1 > $P/ncu_o.log 2>&1; echo "full others rc=$?"
fi

# what the driver runs at round end, on one fresh box
set -u
mkdir -p gpurun_out/drv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/drv/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/drv/smoke.log
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/drv/gputest.log 2>&1; echo "gputest rc=$?"; tail -1 gpurun_out/drv/gputest.log
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/drv/ref.json 2> gpurun_out/drv/ref.err; echo "ref rc=$?"
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/drv/ours.json 2> gpurun_out/drv/ours.err; echo "ours rc=$?"

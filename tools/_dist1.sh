set -u
mkdir -p gpurun_out/q
DIVAS_FORCE_DIST=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 10 --warmup 3 --no-cpu-baseline ${ARGS:-} > gpurun_out/q/dist1.json 2> gpurun_out/q/dist1.err; echo "rc=$?"; tail -5 gpurun_out/q/dist1.err

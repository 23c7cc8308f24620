set -u
P=gpurun_out/q
mkdir -p $P
timeout 300 python tools/profile_step.py --steps 2 > $P/step.log 2>&1; rc=$?; echo "step rc=$rc"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:${KERN:-fuse_pairs} -s 1 -c 1 \
    -o $P/${OUT:-pairs} python tools/profile_step.py --steps 2 > $P/ncu_f.log 2>&1; echo "full rc=$?"

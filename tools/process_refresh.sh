# Turn a tools/refresh_profiles.sh run (gpurun_out/prof_<tag>) into the tracked
# profiles/<tag>_* files and profiles/ncu_traffic.json.  Run here, after the
# gpurun call merged its outputs back.
# usage: bash tools/process_refresh.sh [round-tag]   (default r02)
set -eu
R=${1:-r02}
P=gpurun_out/prof_$R
O=profiles
for f in bench_C1 bench_C2 bench_C3 bench_C5 bench_reference_C3 bench_dist1_C3_C5; do
  tail -1 $P/$f.json > $O/${R}_$f.json
done
cp $P/launches_C3.csv $O/${R}_launches_C3.csv
{
  echo "# $R launch list of the bench step (ncu --metrics gpu__time_duration.sum,dram__bytes_*.sum,smsp__inst_executed.sum --clock-control none on tools/profile_step.py; cold, serialised launches: read the shares)"
  python tools/launch_dram.py $P/launches_C3.csv
} > $O/${R}_launches_C3.txt
{
  echo "# $R ncu --set full --import-source on, fuse_pairs, C3 (one launch of the bench step; marcher inputs; tools/refresh_profiles.sh)"
  python tools/ncu_summary.py report $P/fuse_pairs.ncu-rep
  echo
  echo "## per-function attribution (tools/ncu_funcs.py: warp instructions, lane efficiency, stall samples)"
  python tools/ncu_funcs.py $P/fuse_pairs.ncu-rep fuse_pairs --top 30
} > $O/${R}_ncu_fuse_pairs_C3.txt
{
  echo "# $R ncu --set full of the other step kernels, C3 (tools/refresh_profiles.sh)"
  python tools/ncu_summary.py report $P/others.ncu-rep
} > $O/${R}_ncu_others_C3.txt
{
  echo "# $R ncu --set full of overlay_kernel: project_grid_overlay of the fused C3 grid onto view 31 (tools/profile_overlay.py)"
  python tools/ncu_summary.py report $P/overlay.ncu-rep
} > $O/${R}_ncu_overlay_C3.txt
python tools/make_traffic.py $P/launches_C3.csv C3 "tools/refresh_profiles.sh $R -> $P/launches_C3.csv"
echo "processed $P -> $O/${R}_*"

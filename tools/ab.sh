# A/B of library variants on the bench step; usage: bash tools/ab.sh CONFIG var1 var2 ...
# (a variant name "cur" is the in-tree library)
cfg=$1; shift
for rep in 1 2; do
for v in "$@"; do
  if [ "$v" = cur ]; then unset DIVAS_LIB; else export DIVAS_LIB=/root/repo/_variants/$v.so; fi
  timeout 300 python tools/ab_step.py --config $cfg --iters 30 2>&1 | tail -1 | sed "s/^/$v /"
done
done

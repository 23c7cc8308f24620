# e2e (pinned refine_and_fuse) A/B over library variants and the upload-stream priority
for rep in 1 2; do
for v in cur g2 g4; do
for pr in 0 1; do
  if [ "$v" = cur ]; then unset DIVAS_LIB; else export DIVAS_LIB=/root/repo/_variants/$v.so; fi
  DIVAS_UP_PRIO=$pr E2E_ONLY=1 timeout 300 python tools/_e2e_parts.py 2>&1 | grep "e2e pinned"
done; done; done

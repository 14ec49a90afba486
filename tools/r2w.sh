for env in "X=1" "RT3D_BLOCKS_PER_SM=1" "RT3D_GSZ=4" "RT3D_GSZ=32" "RT3D_TWO_CAND=3" "RT3D_TWO_CAND=0"; do
  echo "== $env"
  env $env timeout 300 python tools/batch_probe.py B 2>&1 | grep -E '"batch": (1|8)'
done

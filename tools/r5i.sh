for g in default 1 4 32; do
  if [ $g = default ]; then BATCHES=1 timeout 300 python tools/batch_probe.py B 2>&1 | tail -1; else RT3D_GSZ=$g BATCHES=1 timeout 300 python tools/batch_probe.py B 2>&1 | tail -1 | sed "s/^/gsz=$g /"; fi
done
RT3D_BLOCKS_PER_SM=3 BATCHES=1 timeout 300 python tools/batch_probe.py B 2>&1 | tail -1 | sed "s/^/bps3 /"
RT3D_ONE_CAND=1 BATCHES=1 timeout 300 python tools/batch_probe.py B 2>&1 | tail -1 | sed "s/^/onecand /"

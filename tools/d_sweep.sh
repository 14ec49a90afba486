#!/bin/bash
# A/B of the stage-kernel switches on config D (and B for reference):
# one JSON line per variant in gpurun_out/d_sweep.jsonl
out=gpurun_out/d_sweep.jsonl
: > $out
for v in "" "RT3D_GSZ=32" "RT3D_GSZ=4" "RT3D_GSZ=3" "RT3D_BLOCKS_PER_SM=1" "RT3D_BLOCKS_PER_SM=3" "RT3D_TWO_CAND=3" "RT3D_ONE_CAND=1"; do
  for c in ${CONFIGS:-D}; do
    line=$(env $v timeout 300 python tools/bench_configs.py 3 $c 2>/dev/null | tail -1)
    echo "{\"variant\": \"$v\", \"result\": ${line:-null}}" >> $out
  done
done

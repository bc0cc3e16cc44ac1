#!/bin/bash
# GPU build_bvh timing + exactness per library variant
out=gpurun_out/bvh_variants.log; rm -f $out
for v in "" bs2048_128 bs1024_128 bs1024_64 bs2048_256 bs512_64; do
  lib=paper_2407_19977_b200/_build/variant_$v/libluxb200.so
  [ -z "$v" ] && lib=paper_2407_19977_b200/_build/libluxb200.so
  echo "== ${v:-default}" >> $out
  LUXB200_LIB=$lib timeout 300 python tools/bvh_build_time.py pushbutton sphere70k >> $out 2>&1
  LUXB200_LIB=$lib timeout 300 python -m pytest tests/test_bvh_gpu.py -q -m gpu -x 2>&1 | tail -1 >> $out
done

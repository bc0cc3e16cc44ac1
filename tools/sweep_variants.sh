#!/bin/bash
# Bench every built library variant (paper_2407_19977_b200/_build/variant_*)
# on the default workload; usage: tools/sweep_variants.sh OUT.jsonl [names...]
out=$1; shift
for v in "$@"; do
  lib=paper_2407_19977_b200/_build/variant_$v/libluxb200.so
  echo "$v" >> "$out"
  LUXB200_LIB=$lib timeout 300 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu >> "$out" 2>> "${out%.jsonl}.err"
done

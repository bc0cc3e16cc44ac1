#!/bin/bash
# Bench the default library under different environment settings;
# usage: tools/sweep_env.sh OUT.jsonl "VAR=a" "VAR=b" ...
out=$1; shift
for e in "$@"; do
  echo "$e" >> "$out"
  env $e timeout 300 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu >> "$out" 2>> "${out%.jsonl}.err"
done

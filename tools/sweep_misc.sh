#!/bin/bash
# lanes / batch-size sweep on the default library
out=$1; rm -f $out
for e in "LT_LANES=2" "LT_LANES=1" "LT_LANES=3" "LT_LANES=4"; do
  echo "$e" >> $out
  env $e timeout 300 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu >> $out 2>> ${out%.jsonl}.err
done
for b in 33554432 50000000; do
  echo "batch=$b" >> $out
  timeout 300 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu --batch-paths $b >> $out 2>> ${out%.jsonl}.err
done

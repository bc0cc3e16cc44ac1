#!/bin/bash
# bench.py on each BASELINE.json config (C1..C5; C5 on one GPU = its whole frame)
out=gpurun_out/configs.jsonl; rm -f $out
run() { echo "$1" >> $out; shift; timeout 600 python bench.py --steps 4 --warmup 3 --cpu-seconds 6 "$@" >> $out 2>> ${out%.jsonl}.err; }
run C1 --workload cornell_c1 --width 64 --height 64 --spp 4 --depth 4
run C2 --workload cornell_c2x --width 512 --height 512 --spp 64 --depth 8
run C3 --workload sphere70k --width 1920 --height 1080 --spp 64 --depth 8
run C4 --workload pushbutton
run C5 --workload pushbutton --width 3840 --height 2160 --spp 1024 --depth 8 --no-e2e --no-cpu

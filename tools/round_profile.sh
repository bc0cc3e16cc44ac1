#!/bin/bash
# One GPU call's worth of evidence for profiles/ (round tag $1):
#   * the driver's bench command (reference arm, then ours) -> ${tag}_bench*.jsonl
#   * C5 (4K, 1024 spp, spp split) on one GPU -> ${tag}_c5.jsonl
#   * the ncu launch list of the same bench command -> ${tag}_launches.csv
#   * the per-level bytes / unit utilisations of the 8 k_trace launches of one
#     whole-frame batch (tools/trace_ncu.py) -> trace_ncu_pushbutton.csv/.log
#   * one --set full capture of the depth-0 / depth-1 k_trace and k_shade
#     launches of a C4 pass -> ${tag}_trace.ncu-rep / ${tag}_shade.ncu-rep
tag=$1
mkdir -p gpurun_out
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 \
  > gpurun_out/${tag}_bench_reference.jsonl 2> gpurun_out/${tag}_bench_reference.err
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 \
  > gpurun_out/${tag}_bench.jsonl 2> gpurun_out/${tag}_bench.err || exit 1
timeout 900 python bench.py --gpus 1 --steps 3 --warmup 1 --config c5 --no-cpu --no-e2e \
  --no-variant > gpurun_out/${tag}_c5.jsonl 2> gpurun_out/${tag}_c5.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e \
  --no-cpu --no-variant > gpurun_out/${tag}_launches.log 2>&1
timeout 1200 python tools/trace_ncu.py capture --workload pushbutton > gpurun_out/${tag}_tncu.log 2>&1
LT_LANES=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_trace -c 2 \
  -f -o gpurun_out/${tag}_trace python tools/profile_pass.py > gpurun_out/${tag}_ncu_trace.log 2>&1
LT_LANES=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_shade -c 2 \
  -f -o gpurun_out/${tag}_shade python tools/profile_pass.py > gpurun_out/${tag}_ncu_shade.log 2>&1
exit 0

#!/bin/bash
# One GPU call's worth of evidence for profiles/: the default bench line,
# the ncu launch list of the same command, and one --set full capture of
# the first two k_trace and k_shade launches (depth 0 and 1) of a C4 pass.
# usage: tools/round_profile.sh TAG
tag=$1
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/${tag}_bench.jsonl 2> gpurun_out/${tag}_bench.err || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu \
  > gpurun_out/${tag}_launches.log 2>&1
LT_LANES=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_trace -c 2 \
  -f -o gpurun_out/${tag}_trace python tools/profile_pass.py > gpurun_out/${tag}_ncu_trace.log 2>&1
LT_LANES=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_shade -c 2 \
  -f -o gpurun_out/${tag}_shade python tools/profile_pass.py > gpurun_out/${tag}_ncu_shade.log 2>&1
exit 0

out=gpurun_out/sweep18.jsonl; rm -f $out
for a in "--bvh-bins 12 --bvh-leaf 4" "--bvh-bins 32 --bvh-leaf 4" "--bvh-bins 32 --bvh-leaf 2" "--bvh-bins 12 --bvh-leaf 2" "--bvh-bins 32 --bvh-leaf 8"; do
  echo "$a" >> $out
  timeout 300 python bench.py --steps 4 --warmup 3 --no-e2e --no-cpu $a >> $out 2>> gpurun_out/sweep18.err
done

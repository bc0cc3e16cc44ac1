#!/bin/bash
# compute-sanitizer over smoke() and a C1 render (64x64, 4 spp, depth 4):
# memcheck (out-of-bounds / misaligned / leaks) and racecheck (shared-memory
# hazards in the persistent trace and shade kernels).  Logs in gpurun_out/.
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
cat > /tmp/lt_c1.py <<'PY'
import sys; sys.path.insert(0, ".")
import workloads, paper_2407_19977_b200 as lb
sc = workloads.scene_by_name("cornell_c1")
r = lb.render_progressive(sc, lb.RenderSettings(samples_per_pixel=4, max_depth=4, seed=7))
print("c1 render ok", r.image.mean())
sc2 = workloads.cornell_box(32, 32, "extended")
r2 = lb.render_progressive(sc2, lb.RenderSettings(samples_per_pixel=2, max_depth=8, seed=3))
print("c2x render ok", r2.image.mean())
PY
for tool in memcheck racecheck; do
  timeout 900 $CS --tool $tool --print-limit 50 python -c "import __graft_entry__ as g; g.smoke()" \
    > gpurun_out/sanitize_${tool}_smoke.log 2>&1; echo "smoke $tool rc=$?" >> gpurun_out/sanitize_${tool}_smoke.log
  timeout 900 $CS --tool $tool --print-limit 50 python /tmp/lt_c1.py \
    > gpurun_out/sanitize_${tool}_c1.log 2>&1; echo "c1 $tool rc=$?" >> gpurun_out/sanitize_${tool}_c1.log
done

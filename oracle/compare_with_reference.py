"""Speed and bit-exactness of the C oracle port against the numba reference on
the same host cores (run here, where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba_cache python oracle/compare_with_reference.py

TEST INFRASTRUCTURE ONLY."""
import os, sys, time
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.path.insert(0, "/root/reference/pkg/src"); sys.path.insert(0, "/root/repo")
import numpy as np
import luxtrace as lx
sys.path.insert(0, "/root/repo/tests/golden")
from make_golden import to_ref_scene
from workloads import scene_by_name
from paper_2407_19977_b200 import camera_pack
from oracle.oracle import OracleScene
W, H, SPP = 240, 135, 8
sc = scene_by_name("pushbutton_ref", width=W, height=H)
ref = to_ref_scene(sc)
t0 = time.perf_counter(); bvh = lx.build_bvh(ref.triangles); print("ref build", time.perf_counter() - t0)
st = lx.RenderSettings(samples_per_pixel=1, max_depth=8, seed=0)
lx.render_progressive(ref, st, bvh=bvh)  # warm JIT
st = lx.RenderSettings(samples_per_pixel=SPP, max_depth=8, seed=0)
r = lx.render_progressive(ref, st, bvh=bvh)
print(f"numba reference: {W*H*SPP/(r.elapsed_ms/1e3)/1e6:.2f} M samples/s ({r.threads_used} threads)")
oc = OracleScene(sc.triangles, bvh, sc.materials, sc.environment)
acc = np.zeros((H, W, 3)); v = np.zeros((H, W), np.int64); iv = np.zeros((H, W), np.int64)
t0 = time.perf_counter()
oc.render_pass(acc, v, iv, 0, SPP, camera_pack(sc.camera), W, H, 0, 8, 3)
dt = time.perf_counter() - t0
print(f"C oracle port:   {W*H*SPP/dt/1e6:.2f} M samples/s ({os.cpu_count()} threads)")
print("images identical:", np.array_equal(acc, r.image))

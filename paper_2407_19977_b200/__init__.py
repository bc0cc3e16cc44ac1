"""paper_2407_19977_b200 -- B200-native Monte-Carlo path tracing of
triangle-mesh scenes with the OpenPBR surface model (arXiv 2407.19977's hot
path), a drop-in for the `luxtrace` reference's render API.

Host code is Python; the hot path is hand-written sm_100a CUDA behind the
C-ABI in include/luxb200.h (built in-tree by `build.py`).  There is no CPU
fallback: compute entry points raise when the library or a GPU is missing.
"""
from .geometry import (DEFAULT_T_MIN, Aabb, Hit, Ray, Triangle, TriangleBuffer, aabb_surface_area,
                       aabb_union, normalize, ray_aabb_intersect, ray_triangle_intersect,
                       triangle_bounds, vec3)
from .material import (OpenPbrParams, emitted_radiance, pack_material_table, pack_materials)
from .scene import (CameraConfig, EnvironmentConfig, SceneDescription, SceneError, camera_pack)
from .rng import PcgState, next_unit_real, pcg_next_u32, pcg_seed, seed_stream
from .bvh import (STACK_SIZE, BuildStats, Bvh, brute_force_intersect_batch, build_bvh,
                  intersect_any, intersect_any_batch, intersect_scene, intersect_scene_batch,
                  intersect_scene_counted, traversal_counts_batch, validate_bvh)
from .bsdf import (BsdfSample, cosine_sample_hemisphere, eval_bsdf, fresnel_schlick, ggx_ndf,
                   ggx_sample_half_vector, pdf_bsdf, sample_bsdf, smith_g2)
from .tonemap import (linear_to_srgb, pbr_neutral_tonemap, quantize_to_u8, srgb_to_linear,
                      tonemap_to_u8, write_linear_dump, write_png)
from ._parallel import set_worker_count, thread_cap
from .device import DeviceScene
from .integrator import (RenderResult, RenderSettings, environment_radiance,
                         generate_camera_ray, render_image, render_pass, render_progressive,
                         trace_radiance, trace_radiance_batch)
from .procgen import bumpy_sphere, bumpy_sphere_glb, icosphere, icosphere_glb
from .harness import (BenchmarkReport, BenchRow, auto_framing_camera, format_ms,
                      load_benchmark_scene, run_benchmark, summarize_runs)
from .ingest import (MaterialMap, RenderConfig, flatten_scene, generate_smooth_normals, load_gltf,
                     load_render_config, load_scene, save_glb, load_device_scene, load_scene_gpu)

__version__ = "0.1.0"

__all__ = [
    "DEFAULT_T_MIN", "Aabb", "Hit", "Ray", "Triangle", "TriangleBuffer", "aabb_surface_area",
    "aabb_union", "normalize", "ray_aabb_intersect", "ray_triangle_intersect",
    "triangle_bounds", "vec3",
    "OpenPbrParams", "emitted_radiance", "pack_material_table", "pack_materials",
    "CameraConfig", "EnvironmentConfig", "SceneDescription", "SceneError", "camera_pack",
    "PcgState", "next_unit_real", "pcg_next_u32", "pcg_seed", "seed_stream",
    "STACK_SIZE", "BuildStats", "Bvh", "brute_force_intersect_batch", "build_bvh",
    "intersect_any", "intersect_any_batch", "intersect_scene", "intersect_scene_batch",
    "intersect_scene_counted", "traversal_counts_batch", "validate_bvh", "DeviceScene",
    "BsdfSample", "cosine_sample_hemisphere", "eval_bsdf", "fresnel_schlick", "ggx_ndf",
    "ggx_sample_half_vector", "pdf_bsdf", "sample_bsdf", "smith_g2",
    "linear_to_srgb", "pbr_neutral_tonemap", "quantize_to_u8", "srgb_to_linear",
    "tonemap_to_u8", "write_linear_dump", "write_png", "set_worker_count", "thread_cap",
    "RenderResult", "RenderSettings", "environment_radiance", "generate_camera_ray",
    "render_image", "render_pass", "render_progressive", "trace_radiance",
    "trace_radiance_batch",
    "bumpy_sphere", "bumpy_sphere_glb", "icosphere", "icosphere_glb",
    "MaterialMap", "RenderConfig", "flatten_scene", "generate_smooth_normals", "load_gltf",
    "load_render_config", "load_scene", "save_glb", "load_device_scene", "load_scene_gpu",
    "BenchRow", "BenchmarkReport", "auto_framing_camera", "format_ms", "load_benchmark_scene",
    "run_benchmark", "summarize_runs",
]

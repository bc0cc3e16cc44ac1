"""Device-side glTF ingest (csrc/lt_ingest.cu) against the
host restatement and the reference's own outputs.

`load_scene_gpu` must return load_scene's SceneDescription bit for bit:
  * on the reference-made fixtures (tests/golden/ingest, expected arrays from
    the reference's load_scene: TRS / matrix / instanced nodes, u8 / u16 /
    u32 indices, strided accessors, generated and explicit normals, a
    degenerate triangle, data-URI buffers);
  * at full size on the C4 pushbutton written as a GLB (1.06 M triangles,
    explicit and generated normals);
  * on a randomised hierarchy (rotations, non-uniform scales, a mirrored
    node, nested and instanced meshes) where numpy's BLAS product fixes the
    rounding of every world coordinate.
`load_device_scene` (the soup never reaches the host) must render exactly
what DeviceScene(load_scene(...)) renders.
"""
from __future__ import annotations

import ctypes as C
import json
import struct

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

DIR = GOLDEN / "ingest"
FIXTURES = ["ico.glb", "ico_normals.glb", "hier.glb", "hier.gltf"]
FIELDS = ["v0", "v1", "v2", "n0", "n1", "n2", "material_index"]


def assert_same_scene(got, want):
    for f in FIELDS:
        a, b = np.asarray(getattr(got.triangles, f)), np.asarray(getattr(want.triangles, f))
        assert a.dtype == b.dtype and a.shape == b.shape, f
        # bit for bit (also tells -0.0 from +0.0)
        assert np.array_equal(a.view(np.uint8), b.view(np.uint8)), \
            f"{f}: {np.count_nonzero(a != b)} of {a.size} values differ"
    assert got.degenerate_dropped == want.degenerate_dropped
    assert got.materials == want.materials


@pytest.mark.parametrize("name", FIXTURES)
def test_load_scene_gpu_matches_reference_fixtures(name):
    from paper_2407_19977_b200.ingest import load_scene_gpu
    z = np.load(GOLDEN / "ingest_expected.npz")
    key = name.replace(".", "_")
    sd = load_scene_gpu(DIR / name, DIR / "config.json")
    for f in FIELDS:
        ref = z[f"{key}__{f}"]
        got = np.asarray(getattr(sd.triangles, f))
        assert got.dtype == ref.dtype, f
        assert np.array_equal(got.view(np.uint8), ref.view(np.uint8)), f
    assert sd.degenerate_dropped == int(z[f"{key}__dropped"])


@pytest.mark.parametrize("normals", [True, False], ids=["normals", "generated"])
def test_load_scene_gpu_pushbutton_bit_exact(tmp_path, normals):
    import workloads
    from paper_2407_19977_b200.ingest import load_scene, load_scene_gpu
    sc = workloads.pushbutton()
    glb, cfg = tmp_path / "pb.glb", tmp_path / "pb.json"
    workloads.write_gltf(sc, glb, cfg, normals=normals)
    want = load_scene(glb, cfg)
    got = load_scene_gpu(glb, cfg)
    assert len(got.triangles.v0) > 1_000_000
    assert_same_scene(got, want)


def _glb(doc: dict, binary: bytes) -> bytes:
    j = json.dumps(doc).encode()
    j += b" " * (-len(j) % 4)
    b = binary + b"\x00" * (-len(binary) % 4)
    return (struct.pack("<III", 0x46546C67, 2, 28 + len(j) + len(b)) +
            struct.pack("<II", len(j), 0x4E4F534A) + j + struct.pack("<II", len(b), 0x004E4942) + b)


def hierarchy_glb(path, seed: int = 3):
    """Randomised node tree over two shared meshes (a bumpy sphere without
    normals, u32 indices; an icosphere with normals, u16 indices)."""
    from paper_2407_19977_b200.procgen import bumpy_sphere, icosphere
    rng = np.random.default_rng(seed)
    pa, ia = bumpy_sphere(60_000)
    pa = np.asarray(pa, np.float32)
    ia = np.asarray(ia, np.uint32).ravel()
    pb, ib = icosphere(3)
    pb = np.asarray(pb, np.float32)
    nb = (pb / np.linalg.norm(pb, axis=1, keepdims=True)).astype(np.float32)
    ib = np.asarray(ib, np.uint16).ravel()
    blobs, views, offs = [pa.tobytes(), ia.tobytes(), pb.tobytes(), nb.tobytes(), ib.tobytes()], [], []
    binary = b""
    for bl in blobs:
        offs.append(len(binary))
        views.append({"buffer": 0, "byteOffset": len(binary), "byteLength": len(bl)})
        binary += bl + b"\x00" * (-len(bl) % 4)
    acc = [{"bufferView": 0, "componentType": 5126, "count": len(pa), "type": "VEC3"},
           {"bufferView": 1, "componentType": 5125, "count": int(ia.size), "type": "SCALAR"},
           {"bufferView": 2, "componentType": 5126, "count": len(pb), "type": "VEC3"},
           {"bufferView": 3, "componentType": 5126, "count": len(nb), "type": "VEC3"},
           {"bufferView": 4, "componentType": 5123, "count": int(ib.size), "type": "SCALAR"}]
    meshes = [{"primitives": [{"attributes": {"POSITION": 0}, "indices": 1, "material": 0}]},
              {"primitives": [{"attributes": {"POSITION": 2, "NORMAL": 3}, "indices": 4,
                               "material": 1},
                              {"attributes": {"POSITION": 2}, "indices": 4}]}]

    def quat():
        q = rng.normal(size=4)
        return [float(x) for x in q / np.linalg.norm(q)]

    def trs():
        return {"translation": [float(x) for x in rng.uniform(-3, 3, 3)], "rotation": quat(),
                "scale": [float(x) for x in rng.uniform(0.3, 2.0, 3)]}

    m = rng.normal(size=(4, 4))
    m[3] = [0, 0, 0, 1]
    m[:3, 0] *= -1.0     # a mirrored (negative-determinant) matrix node
    nodes = [{"children": [1, 2, 4]},
             dict(trs(), mesh=0, children=[3]),
             {"matrix": [float(x) for x in m.T.ravel()], "mesh": 1},
             dict(trs(), mesh=1),
             dict(trs(), children=[5, 6]),
             dict(trs(), mesh=0),
             dict(trs(), mesh=1)]
    doc = {"asset": {"version": "2.0"}, "buffers": [{"byteLength": len(binary)}],
           "bufferViews": views, "accessors": acc, "meshes": meshes, "nodes": nodes,
           "scenes": [{"nodes": [0]}], "scene": 0,
           "materials": [{"name": "shiny_a"},
                         {"name": "b", "pbrMetallicRoughness": {"baseColorFactor": [0.2, 0.5, 0.9, 1],
                                                                "metallicFactor": 0.3}}]}
    path.write_bytes(_glb(doc, binary))


def test_load_scene_gpu_random_hierarchy(tmp_path):
    from paper_2407_19977_b200.ingest import load_scene, load_scene_gpu
    glb = tmp_path / "h.glb"
    for seed in (3, 4):
        hierarchy_glb(glb, seed)
        want = load_scene(glb, DIR / "config.json")
        got = load_scene_gpu(glb, DIR / "config.json")
        assert len(got.triangles.v0) > 100_000
        assert_same_scene(got, want)


def test_load_device_scene_renders_like_the_host_ingest(tmp_path):
    """The resident scene from raw GLB bytes and the host-ingested one give
    bit-identical accumulators (same soup -> same device BVH -> same paths)."""
    import paper_2407_19977_b200 as lb
    from paper_2407_19977_b200.ingest import load_device_scene, load_scene
    from paper_2407_19977_b200.integrator import Accumulator, render_pass_device
    glb = tmp_path / "h.glb"
    hierarchy_glb(glb, 5)
    cfg = tmp_path / "c.json"
    c = json.loads((DIR / "config.json").read_text())
    c["camera"].update(position=[0, 2, 14], width=320, height=240)
    cfg.write_text(json.dumps(c))
    host = load_scene(glb, cfg)
    ds_host = lb.DeviceScene(host)
    ds = load_device_scene(glb, cfg)
    assert ds.n_triangles == len(host.triangles.v0)
    assert ds.degenerate_dropped == host.degenerate_dropped
    assert ds.info["n_nodes"] == ds_host.info["n_nodes"]
    st = lb.RenderSettings(samples_per_pixel=2, max_depth=6, seed=9)
    accs = []
    for d in (ds_host, ds):
        acc = Accumulator(host.camera.width, host.camera.height, d.device)
        render_pass_device(d, host.camera, st, acc, 0, 2)
        accs.append((acc.sum.cpu().numpy(), acc.valid.cpu().numpy()))
    assert np.array_equal(accs[0][0].view(np.uint32), accs[1][0].view(np.uint32))
    assert np.array_equal(accs[0][1], accs[1][1])
    assert accs[0][0].max() > 0.0
    res = lb.render_progressive(ds, lb.RenderSettings(samples_per_pixel=1, max_depth=4))
    assert res.image.shape == (240, 320, 3) and np.isfinite(res.image).all()


def test_device_ingest_errors(tmp_path):
    """All-degenerate geometry is found on the device and raised as the
    reference's SceneError; host-side checks keep the reference's messages;
    a malformed description through the C-ABI fails with LT_ERR_INVALID."""
    from paper_2407_19977_b200 import _lib
    from paper_2407_19977_b200.ingest import load_scene, load_scene_gpu, load_device_scene
    from paper_2407_19977_b200.scene import SceneError
    pos = np.array([[0, 0, 0], [1, 0, 0], [2, 0, 0], [3, 0, 0]], np.float32)  # collinear
    idx = np.array([0, 1, 2, 1, 2, 3], np.uint32)
    doc = {"asset": {"version": "2.0"}, "buffers": [{"byteLength": 72}],
           "bufferViews": [{"buffer": 0, "byteOffset": 0, "byteLength": 48},
                           {"buffer": 0, "byteOffset": 48, "byteLength": 24}],
           "accessors": [{"bufferView": 0, "componentType": 5126, "count": 4, "type": "VEC3"},
                         {"bufferView": 1, "componentType": 5125, "count": 6, "type": "SCALAR"}],
           "meshes": [{"primitives": [{"attributes": {"POSITION": 0}, "indices": 1}]}],
           "nodes": [{"mesh": 0}]}
    glb = tmp_path / "flat.glb"
    glb.write_bytes(_glb(doc, pos.tobytes() + idx.tobytes()))
    for fn in (load_scene, load_scene_gpu, load_device_scene):
        with pytest.raises(SceneError, match="^empty scene$"):
            fn(glb, DIR / "config.json")
    for name in ["badmagic.glb", "truncated.glb", "lines.gltf", "noposition.gltf", "cycle.gltf"]:
        msgs = []
        for fn in (load_scene, load_scene_gpu):
            with pytest.raises(SceneError) as ei:
                fn(DIR / name, DIR / "config.json")
            msgs.append(str(ei.value))
        assert msgs[0] == msgs[1], name
    # C-ABI: an index past the vertex count is caught on the device
    raw = np.frombuffer(pos.tobytes() + np.array([0, 1, 7], np.uint32).tobytes(), np.uint8)
    prim = _lib.GltfPrimitive(pos_buffer=0, pos_stride=12, pos_offset=0, n_vertices=4,
                              nrm_buffer=-1, nrm_stride=12, idx_buffer=0, idx_stride=4,
                              idx_bytes=4, idx_offset=48, n_indices=3)
    inst = _lib.GltfInstance(primitive=0, material=0)
    inst.linear[:] = [1, 0, 0, 0, 1, 0, 0, 0, 1]
    inst.normal_matrix[:] = [1, 0, 0, 0, 1, 0, 0, 0, 1]
    d = _lib.GltfDesc()
    ptrs = (C.POINTER(C.c_uint8) * 1)(raw.ctypes.data_as(C.POINTER(C.c_uint8)))
    sizes = np.array([raw.size], np.int64)
    d.n_buffers, d.buffers, d.buffer_bytes = 1, ptrs, sizes.ctypes.data_as(C.POINTER(C.c_int64))
    d.n_primitives, d.primitives = 1, C.pointer(prim)
    d.n_instances, d.instances = 1, C.pointer(inst)
    out = [np.zeros((1, 3)) for _ in range(6)]
    mat = np.zeros(1, np.int32)
    k, dr = C.c_int64(), C.c_int64()
    dp = C.POINTER(C.c_double)
    rc = _lib.lib().lt_gltf_flatten(C.byref(d), 0, 1, *[a.ctypes.data_as(dp) for a in out],
                                    mat.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(k),
                                    C.byref(dr))
    assert rc == _lib.LT_ERR_INVALID
    assert "index out of range" in _lib.lib().lt_last_error().decode()
    prim.idx_offset = 64    # the index range now overruns the buffer
    rc = _lib.lib().lt_gltf_flatten(C.byref(d), 0, 1, *[a.ctypes.data_as(dp) for a in out],
                                    mat.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(k),
                                    C.byref(dr))
    assert rc == _lib.LT_ERR_INVALID
    assert "outside its buffer" in _lib.lib().lt_last_error().decode()


def random_gltf(rng, path):
    """A random small GLB: 1-3 meshes of 1-2 primitives with u8 / u16 / u32
    or implicit indices, interleaved (strided) or packed float32 positions,
    optional normals, degenerate and empty primitives, and a node tree with
    TRS / matrix / identity nodes, instancing and nested children."""
    blobs, views, accessors = [], [], []
    binary = b""

    def add_view(data: bytes, stride=None):
        nonlocal binary
        v = {"buffer": 0, "byteOffset": len(binary), "byteLength": len(data)}
        if stride:
            v["byteStride"] = stride
        views.append(v)
        binary += data + b"\x00" * (-len(data) % 4)
        return len(views) - 1

    meshes = []
    for _ in range(int(rng.integers(1, 4))):
        prims = []
        for _ in range(int(rng.integers(1, 3))):
            nv = int(rng.integers(3, 40))
            pos = rng.uniform(-2, 2, (nv, 3)).astype(np.float32)
            if rng.uniform() < 0.2:
                pos[1] = pos[0]                      # a degenerate corner pair
            nrm = rng.normal(size=(nv, 3)).astype(np.float32) if rng.uniform() < 0.5 else None
            attrs = {}
            if nrm is not None and rng.uniform() < 0.5:
                v = add_view(np.concatenate([pos, nrm], axis=1).tobytes(), stride=24)
                accessors.append({"bufferView": v, "componentType": 5126, "count": nv,
                                  "type": "VEC3"})
                attrs["POSITION"] = len(accessors) - 1
                accessors.append({"bufferView": v, "byteOffset": 12, "componentType": 5126,
                                  "count": nv, "type": "VEC3"})
                attrs["NORMAL"] = len(accessors) - 1
            else:
                v = add_view(pos.tobytes())
                accessors.append({"bufferView": v, "componentType": 5126, "count": nv,
                                  "type": "VEC3"})
                attrs["POSITION"] = len(accessors) - 1
                if nrm is not None:
                    v = add_view(nrm.tobytes())
                    accessors.append({"bufferView": v, "componentType": 5126, "count": nv,
                                      "type": "VEC3"})
                    attrs["NORMAL"] = len(accessors) - 1
            prim = {"attributes": attrs}
            kind = rng.integers(0, 4)
            if kind < 3:
                nt = int(rng.integers(0, 30))
                idx = rng.integers(0, nv, 3 * nt)
                dt, ct = [(np.uint8, 5121), (np.uint16, 5123), (np.uint32, 5125)][kind]
                v = add_view(idx.astype(dt).tobytes())
                accessors.append({"bufferView": v, "componentType": ct, "count": int(idx.size),
                                  "type": "SCALAR"})
                prim["indices"] = len(accessors) - 1
            elif nv % 3:
                accessors[attrs["POSITION"]]["count"] = nv - nv % 3   # implicit triangles
                if "NORMAL" in attrs:
                    accessors[attrs["NORMAL"]]["count"] = nv - nv % 3
            prims.append(prim)
        meshes.append({"primitives": prims})

    def quat():
        q = rng.normal(size=4)
        return [float(x) for x in q / np.linalg.norm(q)]

    nodes = []
    n_nodes = int(rng.integers(1, 7))
    for i in range(n_nodes):
        node = {}
        r = rng.uniform()
        if r < 0.35:
            node.update(translation=[float(x) for x in rng.uniform(-3, 3, 3)], rotation=quat(),
                        scale=[float(x) for x in rng.uniform(0.2, 2.0, 3)])
        elif r < 0.6:
            m = np.eye(4)
            m[:3, :3] = rng.normal(size=(3, 3))
            m[:3, 3] = rng.uniform(-2, 2, 3)
            node["matrix"] = [float(x) for x in m.T.ravel()]
        if rng.uniform() < 0.8:
            node["mesh"] = int(rng.integers(0, len(meshes)))
        kids = [j for j in range(i + 1, n_nodes) if rng.uniform() < 0.3]
        if kids:
            node["children"] = kids
        nodes.append(node)
    children = {c for n in nodes for c in n.get("children", [])}
    doc = {"asset": {"version": "2.0"}, "buffers": [{"byteLength": len(binary)}],
           "bufferViews": views, "accessors": accessors, "meshes": meshes, "nodes": nodes,
           "scenes": [{"nodes": [i for i in range(n_nodes) if i not in children]}]}
    if path.suffix == ".gltf":
        # a .gltf with its buffer in an external .bin file (the URI resolved
        # next to the document) or inline as a base64 data URI
        if rng.uniform() < 0.5:
            (path.parent / (path.stem + ".bin")).write_bytes(binary)
            doc["buffers"][0]["uri"] = path.stem + ".bin"
        else:
            import base64
            doc["buffers"][0]["uri"] = ("data:application/octet-stream;base64," +
                                        base64.b64encode(binary).decode())
        path.write_text(json.dumps(doc))
    else:
        path.write_bytes(_glb(doc, binary))


def test_device_ingest_fuzz(tmp_path):
    """60 random documents (a third of them .gltf with an external .bin or a
    data-URI buffer): whatever load_scene returns or raises, load_scene_gpu
    returns the same arrays bit for bit or raises the same SceneError."""
    from paper_2407_19977_b200.ingest import load_scene, load_scene_gpu
    rng = np.random.default_rng(2024)
    compared = 0
    for case in range(60):
        glb = tmp_path / (f"r{case}.gltf" if case % 3 == 2 else f"r{case}.glb")
        random_gltf(rng, glb)
        try:
            want = load_scene(glb, DIR / "config.json")
        except Exception as exc:  # noqa: BLE001
            with pytest.raises(type(exc)) as ei:
                load_scene_gpu(glb, DIR / "config.json")
            assert str(ei.value) == str(exc), case
            continue
        got = load_scene_gpu(glb, DIR / "config.json")
        assert_same_scene(got, want)
        compared += 1
    assert compared >= 40

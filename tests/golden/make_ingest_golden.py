"""Ingest fixtures produced by the reference itself.

Run in the build container (the reference is importable there, not on the
GPU box):  NUMBA_CACHE_DIR=/tmp/numba PYTHONPATH=/root/reference/pkg/src \
           python tests/golden/make_ingest_golden.py
Writes tests/golden/ingest/*.{glb,gltf,json} (inputs) and
tests/golden/ingest_expected.npz (the reference's load_scene outputs and
error messages).
"""
import base64
import json
import struct
import sys
from pathlib import Path

import numpy as np

OUT = Path(__file__).resolve().parent / "ingest"
OUT.mkdir(exist_ok=True)

from luxtrace import procgen, scene  # noqa: E402  (the reference)


def glb_bytes(doc: dict, binary: bytes) -> bytes:
    def pad(b, f):
        return b + f * (-len(b) % 4)
    j = pad(json.dumps(doc).encode(), b" ")
    b = pad(binary, b"\x00")
    return (struct.pack("<III", 0x46546C67, 2, 28 + len(j) + len(b)) +
            struct.pack("<II", len(j), 0x4E4F534A) + j + struct.pack("<II", len(b), 0x004E4942) + b)


def hierarchy_doc():
    """Two meshes, TRS / matrix / instanced nodes, u16 and u8 indices,
    generated and explicit normals, a strided accessor, a degenerate triangle."""
    rng = np.random.default_rng(11)
    pa = rng.uniform(-1, 1, (24, 3)).astype(np.float32)
    ia = np.array([[i, (i + 1) % 24, (i + 5) % 24] for i in range(20)] + [[3, 3, 7]], np.uint16)
    pb = rng.uniform(-0.5, 0.5, (9, 3)).astype(np.float32)
    nb = rng.normal(0, 1, (9, 3)).astype(np.float32)
    ib = np.array([[0, 1, 2], [2, 3, 4], [4, 5, 6], [6, 7, 8], [8, 0, 4]], np.uint8)
    # interleaved (strided) positions + normals for mesh B
    inter = np.concatenate([pb, nb], axis=1).astype(np.float32)
    blobs = [pa.tobytes(), ia.tobytes(), inter.tobytes(), ib.tobytes()]
    offs, binary = [], b""
    for bl in blobs:
        offs.append(len(binary))
        binary += bl + b"\x00" * (-len(bl) % 4)
    views = [{"buffer": 0, "byteOffset": offs[0], "byteLength": len(blobs[0])},
             {"buffer": 0, "byteOffset": offs[1], "byteLength": len(blobs[1])},
             {"buffer": 0, "byteOffset": offs[2], "byteLength": len(blobs[2]), "byteStride": 24},
             {"buffer": 0, "byteOffset": offs[3], "byteLength": len(blobs[3])}]
    acc = [{"bufferView": 0, "componentType": 5126, "count": 24, "type": "VEC3"},
           {"bufferView": 1, "componentType": 5123, "count": int(ia.size), "type": "SCALAR"},
           {"bufferView": 2, "componentType": 5126, "count": 9, "type": "VEC3"},
           {"bufferView": 2, "byteOffset": 12, "componentType": 5126, "count": 9, "type": "VEC3"},
           {"bufferView": 3, "componentType": 5121, "count": int(ib.size), "type": "SCALAR"}]
    doc = {
        "asset": {"version": "2.0"},
        "buffers": [{"byteLength": len(binary)}],
        "bufferViews": views, "accessors": acc,
        "materials": [{"name": "shiny_metal", "pbrMetallicRoughness": {
                          "baseColorFactor": [0.9, 0.7, 0.2, 1.0], "metallicFactor": 1.0,
                          "roughnessFactor": 0.25}},
                      {"name": "unbound_plastic", "pbrMetallicRoughness": {
                          "baseColorFactor": [0.1, 0.4, 1.5, 1.0], "metallicFactor": 0.0,
                          "roughnessFactor": 0.6}},
                      {"name": "floor"}],
        "meshes": [{"name": "body", "primitives": [
                       {"attributes": {"POSITION": 0}, "indices": 1, "material": 0},
                       {"attributes": {"POSITION": 0}, "indices": 1, "material": 1}]},
                   {"name": "cap", "primitives": [
                       {"attributes": {"POSITION": 2, "NORMAL": 3}, "indices": 4,
                        "material": 2}]}],
        "nodes": [
            {"name": "root", "translation": [1.0, -2.0, 0.5], "rotation": [0.1, 0.3, -0.2, 0.9],
             "scale": [1.5, 0.75, 2.0], "children": [1, 2]},
            {"name": "arm", "mesh": 0, "matrix": [0.8, 0.1, 0.0, 0.0, -0.1, 0.9, 0.2, 0.0,
                                                  0.0, -0.2, 1.1, 0.0, 0.3, 0.4, -0.5, 1.0],
             "children": [3]},
            {"name": "instance", "mesh": 0, "translation": [4.0, 0.0, 0.0]},
            {"name": "tip", "mesh": 1, "rotation": [0.0, 0.0, 0.7071068, 0.7071068]}],
        "scenes": [{"nodes": [0]}], "scene": 0,
    }
    return doc, binary


def main():
    expected = {}
    # 1. reference writer + loader on the icosphere
    pos, idx = procgen.icosphere(2, 1.0)
    np.savez(OUT / "ico_source.npz", positions=pos, indices=idx)
    procgen.save_glb(OUT / "ico.glb", pos, idx, material_name="shiny_ico")
    procgen.save_glb(OUT / "ico_normals.glb", pos, idx, normals=pos / np.linalg.norm(
        pos, axis=1, keepdims=True))
    # 2. hierarchy: GLB and .gltf with a data-URI buffer
    doc, binary = hierarchy_doc()
    (OUT / "hier.glb").write_bytes(glb_bytes(doc, binary))
    doc2 = json.loads(json.dumps(doc))
    doc2["buffers"] = [{"byteLength": len(binary), "uri": "data:application/octet-stream;base64,"
                        + base64.b64encode(binary).decode()}]
    (OUT / "hier.gltf").write_text(json.dumps(doc2))
    # 3. config
    cfg = {"camera": {"position": [0, 1, 6], "look_at": [0, 0, 0], "vertical_fov_deg": 40,
                      "width": 64, "height": 48},
           "environment": {"type": "gradient", "zenith": [0.2, 0.3, 0.8],
                           "horizon": [0.9, 0.8, 0.7]},
           "materials": {"shiny*": {"base_metalness": 1.0, "specular_roughness": 0.1,
                                    "base_color": [0.95, 0.9, 0.8]},
                         "floor": {"base_color": [0.5, 0.5, 0.5], "specular_weight": 0.0}},
           "default_material": {"base_color": [0.3, 0.6, 0.3]}}
    (OUT / "config.json").write_text(json.dumps(cfg))
    for name in ["ico.glb", "ico_normals.glb", "hier.glb", "hier.gltf"]:
        sd = scene.load_scene(OUT / name, OUT / "config.json")
        t = sd.triangles
        key = name.replace(".", "_")
        for f in ["v0", "v1", "v2", "n0", "n1", "n2", "material_index"]:
            expected[f"{key}__{f}"] = getattr(t, f)
        expected[f"{key}__dropped"] = np.array(sd.degenerate_dropped)
        fields = ["base_weight", "base_color", "base_metalness", "specular_weight",
                  "specular_color", "specular_roughness", "specular_ior", "emission_luminance",
                  "emission_color"]
        expected[f"{key}__materials"] = np.array(
            [np.concatenate([np.ravel(getattr(m, f)) for f in fields]) for m in sd.materials])
    # 4. malformed inputs: the reference's messages
    bad = {
        "truncated.glb": b"glTF\x02\x00",
        "badmagic.glb": b"glTX" + struct.pack("<II", 2, 12),
        "lines.gltf": json.dumps({"asset": {"version": "2.0"}, "meshes": [{"primitives": [
            {"attributes": {"POSITION": 0}, "mode": 1}]}]}).encode(),
        "noposition.gltf": json.dumps({"asset": {"version": "2.0"}, "meshes": [{"primitives": [
            {"attributes": {}}]}]}).encode(),
        "cycle.gltf": json.dumps({"asset": {"version": "2.0"}, "nodes": [
            {"children": [1]}, {"children": [0]}], "scenes": [{"nodes": [0]}]}).encode(),
        "bad_config.json": json.dumps({"camera": {"position": [0, 0, 1]}}).encode(),
    }
    msgs = []
    for name, data in bad.items():
        (OUT / name).write_bytes(data)
        try:
            if name.endswith(".json"):
                scene.load_render_config(OUT / name)
            else:
                doc_ = scene.load_gltf(OUT / name)
                scene.flatten_scene(doc_, scene.MaterialMap(), scene.CameraConfig(
                    position=(0, 0, 1), look_at=(0, 0, 0)), scene.EnvironmentConfig.uniform(
                    (0, 0, 0)))
            msgs.append((name, "no error"))
        except Exception as exc:  # noqa: BLE001
            msgs.append((name, f"{type(exc).__name__}: {exc}".replace(str(OUT), "<DIR>")))
    expected["errors"] = np.array([f"{n}\t{m}" for n, m in msgs])
    np.savez_compressed(OUT.parent / "ingest_expected.npz", **expected)
    for n, m in msgs:
        print(n, "->", m)


if __name__ == "__main__":
    sys.exit(main())

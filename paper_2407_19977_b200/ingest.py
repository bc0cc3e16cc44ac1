"""Scene ingest: the render-config document, the glTF 2.0
subset reader, node-hierarchy flattening and the single-mesh GLB writer of
the `luxtrace` reference (scene.py:44-603, procgen.py:117-190), restated so
`load_scene(gltf, config)` yields the same `SceneDescription` -- the same
float64 triangle arrays bit for bit (the world transform, smooth normals,
degenerate filter and normalisation are the same numpy operations in the
same order) and the same `SceneError` messages.

Host code: ingest produces the arrays `DeviceScene` uploads; the GPU work
starts at `lt_scene_create`.
"""
from __future__ import annotations

import base64
import json
import math
import struct
from dataclasses import dataclass, field
from pathlib import Path
from urllib.parse import unquote

import numpy as np

from .geometry import TriangleBuffer
from .material import OpenPbrParams
from .scene import CameraConfig, EnvironmentConfig, SceneDescription, SceneError

DEGENERATE_AREA_SCALE = 1e-12   # scene.py:29: area threshold / extent^2

GLB_MAGIC = 0x46546C67           # "glTF"
CHUNK_JSON = 0x4E4F534A
CHUNK_BIN = 0x004E4942
COMPONENT_DTYPE = {5120: np.int8, 5121: np.uint8, 5122: np.int16, 5123: np.uint16,
                   5125: np.uint32, 5126: np.float32}
TYPE_WIDTH = {"SCALAR": 1, "VEC2": 2, "VEC3": 3, "VEC4": 4, "MAT4": 16}
INDEX_COMPONENTS = (5121, 5123, 5125)


# ------------------------------------------------------------ render config

@dataclass
class MaterialMap:
    """Ordered (pattern -> parameters) bindings; a pattern is an exact glTF
    material name or a prefix ending in one '*'; the first match wins
    (scene.py:112-137)."""

    entries: list = field(default_factory=list)
    default: OpenPbrParams = field(default_factory=OpenPbrParams)

    def __post_init__(self) -> None:
        for pattern, _ in self.entries:
            n_star = pattern.count("*")
            if n_star > 1 or (n_star == 1 and not pattern.endswith("*")):
                raise SceneError(f"material pattern {pattern!r}: only a single trailing '*' "
                                 "wildcard is supported")

    def resolve(self, name: str):
        for pattern, params in self.entries:
            matched = name.startswith(pattern[:-1]) if pattern.endswith("*") else name == pattern
            if matched:
                return params
        return None


@dataclass
class RenderConfig:
    camera: CameraConfig
    environment: EnvironmentConfig
    materials: MaterialMap


def _material_params(spec, where: str) -> OpenPbrParams:
    """A material object of the config (scene.py:147-164)."""
    if not isinstance(spec, dict):
        raise SceneError(f"{where}: material parameters must be an object, "
                         f"got {type(spec).__name__}")
    fields = OpenPbrParams.__dataclass_fields__
    kwargs = {}
    for key, value in spec.items():
        if key not in fields:
            raise SceneError(f"{where}: unknown material parameter {key!r}")
        if key == "base_color" or key.endswith("_color"):
            if not (isinstance(value, (list, tuple)) and len(value) == 3):
                raise SceneError(f"{where}: {key} must be a list of three numbers")
            kwargs[key] = tuple(float(c) for c in value)
        else:
            kwargs[key] = float(value)
    try:
        return OpenPbrParams(**kwargs)
    except ValueError as exc:
        raise SceneError(f"{where}: {exc}") from exc


def load_render_config(path) -> RenderConfig:
    """The JSON render config: camera, environment, material map
    (scene.py:167-218)."""
    path = Path(path)
    if not path.is_file():
        raise SceneError(f"config file not found: {path}")
    try:
        doc = json.loads(path.read_text())
    except json.JSONDecodeError as exc:
        raise SceneError(f"malformed config JSON in {path}: {exc}") from exc
    if not isinstance(doc, dict):
        raise SceneError(f"config root must be an object: {path}")
    allowed = {"camera", "environment", "materials", "default_material"}
    extra = set(doc) - allowed
    if extra:
        raise SceneError(f"unknown config keys {sorted(extra)}; expected a subset of "
                         f"{sorted(allowed)}")
    for section in ("camera", "environment"):
        if section not in doc:
            raise SceneError(f"config is missing the required '{section}' section")

    cam = doc["camera"]
    if not isinstance(cam, dict) or "position" not in cam or "look_at" not in cam:
        raise SceneError("camera section must contain 'position' and 'look_at'")
    camera = CameraConfig(position=cam["position"], look_at=cam["look_at"],
                          up=cam.get("up", (0.0, 1.0, 0.0)),
                          vertical_fov_deg=float(cam.get("vertical_fov_deg", 45.0)),
                          width=int(cam.get("width", 512)), height=int(cam.get("height", 512)))

    env = doc["environment"]
    if not isinstance(env, dict) or "type" not in env:
        raise SceneError("environment section must contain a 'type'")
    kind = env["type"]
    if kind == "uniform":
        if "radiance" not in env:
            raise SceneError("uniform environment requires 'radiance'")
        environment = EnvironmentConfig.uniform(env["radiance"])
    elif kind == "gradient":
        if "zenith" not in env or "horizon" not in env:
            raise SceneError("gradient environment requires 'zenith' and 'horizon'")
        environment = EnvironmentConfig.gradient(env["zenith"], env["horizon"])
    else:
        raise SceneError(f"environment type must be 'uniform' or 'gradient', got {kind!r}")

    bindings = [(pattern, _material_params(spec, f"materials[{pattern!r}]"))
                for pattern, spec in doc.get("materials", {}).items()]
    default = (_material_params(doc["default_material"], "default_material")
               if "default_material" in doc else OpenPbrParams())
    return RenderConfig(camera, environment, MaterialMap(bindings, default))


# ------------------------------------------------------------ glTF document

@dataclass
class GltfPrimitive:
    positions: np.ndarray            # (m, 3) float64 (widened float32)
    normals: np.ndarray | None
    indices: np.ndarray              # (3k,) int64
    material_name: str | None
    material_fallback: OpenPbrParams | None


@dataclass
class GltfMesh:
    name: str
    primitives: list


@dataclass
class GltfNode:
    name: str
    matrix: np.ndarray               # local 4x4
    mesh: int | None
    children: list


@dataclass
class GltfDocument:
    meshes: list
    nodes: list
    roots: list


class _GltfReader:
    """One glTF / GLB file: container, buffers, accessors, node matrices
    (scene.py:251-380)."""

    def __init__(self, path: Path):
        self.path = path
        raw = path.read_bytes()
        binary = None
        if raw[:4] == b"glTF":
            doc, binary = self._unpack_glb(raw)
        else:
            try:
                doc = json.loads(raw)
            except json.JSONDecodeError as exc:
                raise SceneError(f"{path}: malformed glTF JSON: {exc}") from exc
        if not isinstance(doc, dict):
            raise SceneError(f"{path}: glTF root must be a JSON object")
        self.doc = doc
        self.buffers = self._load_buffers(binary)

    def _unpack_glb(self, raw: bytes):
        path = self.path
        if len(raw) < 12:
            raise SceneError(f"{path}: truncated GLB header")
        magic, version, total = struct.unpack_from("<III", raw, 0)
        if magic != GLB_MAGIC:
            raise SceneError(f"{path}: not a GLB container (bad magic)")
        if version != 2:
            raise SceneError(f"{path}: unsupported GLB version {version}")
        doc = binary = None
        pos = 12
        end = min(total, len(raw))
        while pos + 8 <= end:
            size, kind = struct.unpack_from("<II", raw, pos)
            pos += 8
            if pos + size > len(raw):
                raise SceneError(f"{path}: GLB chunk at byte {pos - 8} overruns the file")
            body = raw[pos:pos + size]
            pos += size
            if kind == CHUNK_JSON:
                try:
                    doc = json.loads(body)
                except json.JSONDecodeError as exc:
                    raise SceneError(f"{path}: malformed glTF JSON chunk: {exc}") from exc
            elif kind == CHUNK_BIN:
                binary = body
        if doc is None:
            raise SceneError(f"{path}: GLB container has no JSON chunk")
        return doc, binary

    def _load_buffers(self, glb_binary):
        out = []
        for i, spec in enumerate(self.doc.get("buffers", [])):
            uri = spec.get("uri")
            if uri is None:
                if glb_binary is None:
                    raise SceneError(f"buffer {i}: no URI and no GLB binary chunk")
                data = glb_binary
            elif uri.startswith("data:"):
                try:
                    data = base64.b64decode(uri.split(",", 1)[1])
                except (ValueError, IndexError, base64.binascii.Error) as exc:
                    raise SceneError(f"buffer {i}: malformed data URI: {exc}") from exc
            else:
                target = self.path.parent / unquote(uri)
                if not target.is_file():
                    raise SceneError(f"buffer {i}: file not found: {target}")
                data = target.read_bytes()
            length = spec.get("byteLength", len(data))
            if len(data) < length:
                raise SceneError(f"buffer {i}: expected {length} bytes, got {len(data)}")
            out.append(data[:length])
        return out

    def accessor_spec(self, idx) -> dict:
        acc = self.doc.get("accessors", [])
        return acc[idx] if idx < len(acc) else {}

    def read(self, idx: int) -> np.ndarray:
        """(count, width) array of an accessor, strided views gathered."""
        accessors = self.doc.get("accessors", [])
        if not 0 <= idx < len(accessors):
            raise SceneError(f"accessor {idx} does not exist")
        acc = accessors[idx]
        if "sparse" in acc:
            raise SceneError(f"accessor {idx}: sparse accessors are not supported")
        ctype = acc.get("componentType")
        if ctype not in COMPONENT_DTYPE:
            raise SceneError(f"accessor {idx}: unsupported componentType {ctype}")
        if acc.get("type") not in TYPE_WIDTH:
            raise SceneError(f"accessor {idx}: unsupported type {acc.get('type')!r}")
        dt = np.dtype(COMPONENT_DTYPE[ctype])
        width = TYPE_WIDTH[acc["type"]]
        count = int(acc.get("count", 0))
        if count == 0:
            return np.zeros((0, width), dtype=dt)
        view_idx = acc.get("bufferView")
        if view_idx is None:
            return np.zeros((count, width), dtype=dt)
        views = self.doc.get("bufferViews", [])
        if not 0 <= view_idx < len(views):
            raise SceneError(f"accessor {idx}: bufferView {view_idx} does not exist")
        view = views[view_idx]
        buf_idx = view.get("buffer", 0)
        if not 0 <= buf_idx < len(self.buffers):
            raise SceneError(f"accessor {idx}: buffer {buf_idx} does not exist")
        raw = self.buffers[buf_idx]
        elem = dt.itemsize * width
        stride = int(view.get("byteStride", 0)) or elem
        first = int(view.get("byteOffset", 0)) + int(acc.get("byteOffset", 0))
        last = first + stride * (count - 1) + elem
        view_end = int(view.get("byteOffset", 0)) + int(view.get("byteLength", len(raw)))
        if last > len(raw) or last > view_end:
            raise SceneError(f"accessor {idx}: data range [{first}, {last}) overruns its "
                             "buffer view")
        if stride == elem:
            return np.frombuffer(raw, dtype=dt, count=count * width, offset=first).reshape(
                count, width)
        rows = np.lib.stride_tricks.as_strided(np.frombuffer(raw, dtype=np.uint8)[first:],
                                               shape=(count, elem), strides=(stride, 1))
        return rows.copy().view(dt).reshape(count, width)


def node_matrix(node: dict, index: int) -> np.ndarray:
    """Local transform: the column-major `matrix`, or T @ R @ S from TRS
    (scene.py:354-381)."""
    if "matrix" in node:
        m = np.asarray(node["matrix"], dtype=np.float64)
        if m.size != 16:
            raise SceneError(f"node {index}: matrix must have 16 entries")
        return m.reshape(4, 4, order="F")
    m = np.eye(4)
    if "scale" in node:
        m[0, 0], m[1, 1], m[2, 2] = (float(v) for v in node["scale"])
    if "rotation" in node:
        qx, qy, qz, qw = (float(v) for v in node["rotation"])
        norm = math.sqrt(qx * qx + qy * qy + qz * qz + qw * qw)
        if norm == 0.0:
            raise SceneError(f"node {index}: zero-length rotation quaternion")
        qx, qy, qz, qw = qx / norm, qy / norm, qz / norm, qw / norm
        rot = np.eye(4)
        rot[:3, :3] = np.array([
            [1 - 2 * (qy * qy + qz * qz), 2 * (qx * qy - qz * qw), 2 * (qx * qz + qy * qw)],
            [2 * (qx * qy + qz * qw), 1 - 2 * (qx * qx + qz * qz), 2 * (qy * qz - qx * qw)],
            [2 * (qx * qz - qy * qw), 2 * (qy * qz + qx * qw), 1 - 2 * (qx * qx + qy * qy)],
        ])
        m = rot @ m
    if "translation" in node:
        tr = np.eye(4)
        tr[:3, 3] = [float(v) for v in node["translation"]]
        m = tr @ m
    return m


def _primitive(reader: _GltfReader, prim: dict, where: str, materials: list) -> GltfPrimitive:
    mode = prim.get("mode", 4)
    if mode != 4:
        raise SceneError(f"{where}: unsupported primitive mode {mode}; only TRIANGLES (4) is "
                         "supported")
    attrs = prim.get("attributes", {})
    if "POSITION" not in attrs:
        raise SceneError(f"{where}: missing POSITION attribute")
    spec = reader.accessor_spec(attrs["POSITION"])
    if spec.get("componentType") != 5126 or spec.get("type") != "VEC3":
        raise SceneError(f"{where}: POSITION must be a float32 VEC3 accessor")
    positions = reader.read(attrs["POSITION"]).astype(np.float64)
    normals = None
    if "NORMAL" in attrs:
        spec = reader.doc["accessors"][attrs["NORMAL"]]
        if spec.get("componentType") != 5126 or spec.get("type") != "VEC3":
            raise SceneError(f"{where}: NORMAL must be a float32 VEC3 accessor")
        normals = reader.read(attrs["NORMAL"]).astype(np.float64)
        if normals.shape != positions.shape:
            raise SceneError(f"{where}: NORMAL count differs from POSITION count")
    if "indices" in prim:
        spec = reader.accessor_spec(prim["indices"])
        if spec.get("componentType") not in INDEX_COMPONENTS or spec.get("type") != "SCALAR":
            raise SceneError(f"{where}: indices must be a scalar u8/u16/u32 accessor")
        indices = reader.read(prim["indices"]).astype(np.int64).ravel()
    else:
        indices = np.arange(positions.shape[0], dtype=np.int64)
    if indices.size % 3 != 0:
        raise SceneError(f"{where}: index count {indices.size} is not a multiple of 3")
    if indices.size and (indices.min() < 0 or indices.max() >= positions.shape[0]):
        raise SceneError(f"{where}: index out of range")
    name = fallback = None
    if "material" in prim:
        m_idx = prim["material"]
        if not 0 <= m_idx < len(materials):
            raise SceneError(f"{where}: material {m_idx} does not exist")
        mat = materials[m_idx]
        name = mat.get("name", f"material_{m_idx}")
        pbr = mat.get("pbrMetallicRoughness", {})
        base = pbr.get("baseColorFactor", [1.0, 1.0, 1.0, 1.0])

        def unit(x):
            return min(max(float(x), 0.0), 1.0)
        fallback = OpenPbrParams(base_color=tuple(unit(c) for c in base[:3]),
                                 base_metalness=unit(pbr.get("metallicFactor", 1.0)),
                                 specular_roughness=unit(pbr.get("roughnessFactor", 1.0)))
    return GltfPrimitive(positions, normals, indices, name, fallback)


def load_gltf(path) -> GltfDocument:
    """Mesh-space geometry plus the node hierarchy of a .gltf / .glb file
    (scene.py:384-490)."""
    path = Path(path)
    if not path.is_file():
        raise SceneError(f"scene file not found: {path}")
    reader = _GltfReader(path)
    doc = reader.doc
    materials = doc.get("materials", [])
    meshes = []
    for mi, mesh in enumerate(doc.get("meshes", [])):
        name = mesh.get("name", f"mesh_{mi}")
        prims = [_primitive(reader, prim, f"mesh {mi} ({name!r}) primitive {pi}", materials)
                 for pi, prim in enumerate(mesh.get("primitives", []))]
        meshes.append(GltfMesh(name, prims))
    nodes = []
    for ni, node in enumerate(doc.get("nodes", [])):
        mesh_idx = node.get("mesh")
        if mesh_idx is not None and not 0 <= mesh_idx < len(meshes):
            raise SceneError(f"node {ni}: mesh {mesh_idx} does not exist")
        nodes.append(GltfNode(node.get("name", f"node_{ni}"), node_matrix(node, ni), mesh_idx,
                              list(node.get("children", []))))
    scenes = doc.get("scenes", [])
    if scenes:
        which = doc.get("scene", 0)
        if not 0 <= which < len(scenes):
            raise SceneError(f"default scene {which} does not exist")
        roots = list(scenes[which].get("nodes", []))
    else:
        children = {c for n in nodes for c in n.children}
        roots = [i for i in range(len(nodes)) if i not in children]
    for r in roots:
        if not 0 <= r < len(nodes):
            raise SceneError(f"scene references node {r} which does not exist")
    return GltfDocument(meshes, nodes, roots)


# ------------------------------------------------------------ flattening

def generate_smooth_normals(positions: np.ndarray, indices: np.ndarray) -> np.ndarray:
    """Area-weighted vertex normals (scene.py:493-508)."""
    a, b, c = (positions[indices[k::3]] for k in range(3))
    face = np.cross(b - a, c - a)          # |face| = 2 * area
    acc = np.zeros_like(positions)
    for k in range(3):
        np.add.at(acc, indices[k::3], face)
    length = np.linalg.norm(acc, axis=1, keepdims=True)
    flat = length[:, 0] == 0.0
    acc[flat] = (0.0, 0.0, 1.0)
    length[flat] = 1.0
    return acc / length


def flatten_scene(doc: GltfDocument, materials: MaterialMap, camera: CameraConfig,
                  environment: EnvironmentConfig) -> SceneDescription:
    """World-space triangle soup: node transforms baked in, materials
    resolved (config name -> glTF fallback -> default), degenerate triangles
    dropped (scene.py:519-596)."""
    parts = []
    table: dict = {}
    params_list: list = []

    def material_slot(params) -> int:
        if params not in table:
            table[params] = len(params_list)
            params_list.append(params)
        return table[params]

    def walk(idx: int, parent: np.ndarray, path: tuple) -> None:
        if idx in path:
            raise SceneError(f"node {idx}: cycle in node hierarchy")
        node = doc.nodes[idx]
        world = parent @ node.matrix
        if node.mesh is not None:
            linear = world[:3, :3]
            if float(np.linalg.det(linear)) == 0.0:
                raise SceneError(f"node {idx} ({node.name!r}): singular transform")
            to_normals = np.linalg.inv(linear).T
            for prim in doc.meshes[node.mesh].primitives:
                world_pos = prim.positions @ linear.T + world[:3, 3]
                local_n = prim.normals if prim.normals is not None else \
                    generate_smooth_normals(prim.positions, prim.indices)
                world_n = local_n @ to_normals.T
                params = materials.resolve(prim.material_name) if prim.material_name else None
                if params is None:
                    params = prim.material_fallback
                if params is None:
                    params = materials.default
                slot = material_slot(params)
                ix = prim.indices
                parts.append(tuple(world_pos[ix[k::3]] for k in range(3)) +
                             tuple(world_n[ix[k::3]] for k in range(3)) + (slot,))
        for child in node.children:
            walk(child, world, path + (idx,))

    for root in doc.roots:
        walk(root, np.eye(4), ())
    if not parts or sum(p[0].shape[0] for p in parts) == 0:
        raise SceneError("empty scene")
    v0, v1, v2, n0, n1, n2 = (np.vstack([p[k] for p in parts]) for k in range(6))
    mat = np.concatenate([np.full(p[0].shape[0], p[6], dtype=np.int32) for p in parts])

    corners = np.vstack([v0, v1, v2])
    extent = float(np.max(corners.max(axis=0) - corners.min(axis=0)))
    areas = 0.5 * np.linalg.norm(np.cross(v1 - v0, v2 - v0), axis=1)
    keep = areas > DEGENERATE_AREA_SCALE * extent * extent
    dropped = int(np.count_nonzero(~keep))
    if not np.any(keep):
        raise SceneError("empty scene")

    def unit_rows(a):
        length = np.linalg.norm(a, axis=1, keepdims=True)
        length[length == 0.0] = 1.0
        return a / length

    tris = TriangleBuffer(v0[keep], v1[keep], v2[keep], unit_rows(n0[keep]),
                          unit_rows(n1[keep]), unit_rows(n2[keep]), mat[keep])
    return SceneDescription(tris, params_list, camera, environment, dropped)


def load_scene(scene_path, config_path) -> SceneDescription:
    """glTF file + render config -> SceneDescription (scene.py:599-603)."""
    config = load_render_config(config_path)
    return flatten_scene(load_gltf(scene_path), config.materials, config.camera,
                         config.environment)


# ------------------------------------------------------------ GLB writer

def save_glb(path, positions, indices, normals=None, material_name=None) -> None:
    """Single-mesh GLB (float32 positions, optional normals, u32 indices; one
    node, one scene) byte-identical to the reference writer
    (procgen.py:117-190)."""
    positions = np.ascontiguousarray(positions, dtype=np.float32)
    indices = np.ascontiguousarray(indices, dtype=np.uint32).ravel()
    if positions.ndim != 2 or positions.shape[1] != 3:
        raise ValueError("positions must have shape (n, 3)")
    if indices.size % 3 != 0:
        raise ValueError("index count must be a multiple of 3")
    if normals is not None:
        normals = np.ascontiguousarray(normals, dtype=np.float32)
        if normals.shape != positions.shape:
            raise ValueError("normals must match positions in shape")

    def padded(data: bytes, fill: bytes) -> bytes:
        return data + fill * (-len(data) % 4)

    blobs = [positions.tobytes()] + ([normals.tobytes()] if normals is not None else []) + \
        [indices.tobytes()]
    views, offset = [], 0
    for blob in blobs:
        views.append({"buffer": 0, "byteOffset": offset, "byteLength": len(blob)})
        offset += len(padded(blob, b"\x00"))
    binary = b"".join(padded(b, b"\x00") for b in blobs)
    accessors = [{"bufferView": 0, "componentType": 5126, "count": int(positions.shape[0]),
                  "type": "VEC3", "min": [float(v) for v in positions.min(axis=0)],
                  "max": [float(v) for v in positions.max(axis=0)]}]
    attributes = {"POSITION": 0}
    if normals is not None:
        accessors.append({"bufferView": 1, "componentType": 5126,
                          "count": int(normals.shape[0]), "type": "VEC3"})
        attributes["NORMAL"] = 1
    accessors.append({"bufferView": len(views) - 1, "componentType": 5125,
                      "count": int(indices.size), "type": "SCALAR"})
    primitive = {"attributes": attributes, "indices": len(accessors) - 1, "mode": 4}
    doc = {"asset": {"version": "2.0", "generator": "luxtrace.procgen"},
           "buffers": [{"byteLength": len(binary)}], "bufferViews": views,
           "accessors": accessors, "meshes": [{"name": "mesh_0", "primitives": [primitive]}],
           "nodes": [{"mesh": 0, "name": "node_0"}], "scenes": [{"nodes": [0]}], "scene": 0}
    if material_name is not None:
        doc["materials"] = [{"name": material_name, "pbrMetallicRoughness": {
            "baseColorFactor": [0.8, 0.8, 0.8, 1.0], "metallicFactor": 0.0,
            "roughnessFactor": 0.5}}]
        primitive["material"] = 0
    json_chunk = padded(json.dumps(doc, separators=(",", ":")).encode(), b" ")
    bin_chunk = padded(binary, b"\x00")
    with open(path, "wb") as fh:
        fh.write(struct.pack("<III", GLB_MAGIC, 2, 12 + 8 + len(json_chunk) + 8 +
                             len(bin_chunk)))
        fh.write(struct.pack("<II", len(json_chunk), CHUNK_JSON) + json_chunk)
        fh.write(struct.pack("<II", len(bin_chunk), CHUNK_BIN) + bin_chunk)

"""Scene ingest: the render-config document, the glTF 2.0
subset reader, node-hierarchy flattening and the single-mesh GLB writer of
the `luxtrace` reference (scene.py:44-603, procgen.py:117-190), restated so
`load_scene(gltf, config)` yields the same `SceneDescription` -- the same
float64 triangle arrays bit for bit (the world transform, smooth normals,
degenerate filter and normalisation are the same numpy operations in the
same order) and the same `SceneError` messages.

Two ways to the device:
  * `load_scene` (host, numpy) -> SceneDescription -> `DeviceScene` uploads
    the float64 soup (the reference's path);
  * `load_device_scene` / `load_scene_gpu` (lt_ingest.cu): the host parses
    the JSON, validates the accessors and walks the nodes (cheap); the GLB's
    raw float32 / integer bytes are uploaded once and the device decodes
    them, generates smooth normals, applies the transforms, filters
    degenerates and normalises -- the same float64 arithmetic in the same
    order, so the arrays equal load_scene's bit for bit -- and (for
    load_device_scene) builds the BVH and the render layout without the
    soup ever reaching the host.
"""
from __future__ import annotations

import base64
import contextlib
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

    def locate(self, idx: int) -> "_Located":
        """Where an accessor's elements lie (validated as read() validates)."""
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
        elem = dt.itemsize * width
        count = int(acc.get("count", 0))
        if count == 0:
            return _Located(None, 0, elem, 0, width, dt)
        view_idx = acc.get("bufferView")
        if view_idx is None:
            return _Located(None, 0, elem, count, width, dt)     # all zeros
        views = self.doc.get("bufferViews", [])
        if not 0 <= view_idx < len(views):
            raise SceneError(f"accessor {idx}: bufferView {view_idx} does not exist")
        view = views[view_idx]
        buf_idx = view.get("buffer", 0)
        if not 0 <= buf_idx < len(self.buffers):
            raise SceneError(f"accessor {idx}: buffer {buf_idx} does not exist")
        raw = self.buffers[buf_idx]
        stride = int(view.get("byteStride", 0)) or elem
        first = int(view.get("byteOffset", 0)) + int(acc.get("byteOffset", 0))
        last = first + stride * (count - 1) + elem
        view_end = int(view.get("byteOffset", 0)) + int(view.get("byteLength", len(raw)))
        if last > len(raw) or last > view_end:
            raise SceneError(f"accessor {idx}: data range [{first}, {last}) overruns its "
                             "buffer view")
        return _Located(raw, first, stride, count, width, dt)

    def read(self, idx: int) -> np.ndarray:
        """(count, width) array of an accessor, strided views gathered."""
        return self.locate(idx).array()


@dataclass
class _Located:
    """An accessor's elements: `count` rows of `width` x `dtype`, `stride`
    bytes apart from byte `first` of `data` (None: all zeros)."""
    data: bytes | None
    first: int
    stride: int
    count: int
    width: int
    dtype: np.dtype

    def array(self) -> np.ndarray:
        dt, width, count = self.dtype, self.width, self.count
        if self.data is None:
            return np.zeros((count, width), dtype=dt)
        elem = dt.itemsize * width
        if self.stride == elem:
            return np.frombuffer(self.data, dtype=dt, count=count * width,
                                 offset=self.first).reshape(count, width)
        rows = np.lib.stride_tricks.as_strided(
            np.frombuffer(self.data, dtype=np.uint8)[self.first:], shape=(count, elem),
            strides=(self.stride, 1))
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


@dataclass
class GltfPrimitiveRef:
    """A primitive as located accessors (the device ingest's input): no
    float64 widening on the host."""
    positions: _Located
    normals: _Located | None
    indices: _Located | None          # None: 0 .. n-1
    n_indices: int
    material_name: str | None
    material_fallback: OpenPbrParams | None


def _primitive_ref(reader: _GltfReader, prim: dict, where: str, materials: list):
    """The checks of scene.py:251-351 in the reference's order; returns the
    located primitive and its index values (None when implicit)."""
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
    positions = reader.locate(attrs["POSITION"])
    normals = None
    if "NORMAL" in attrs:
        spec = reader.doc["accessors"][attrs["NORMAL"]]
        if spec.get("componentType") != 5126 or spec.get("type") != "VEC3":
            raise SceneError(f"{where}: NORMAL must be a float32 VEC3 accessor")
        normals = reader.locate(attrs["NORMAL"])
        if normals.count != positions.count:
            raise SceneError(f"{where}: NORMAL count differs from POSITION count")
    values = indices = None
    if "indices" in prim:
        spec = reader.accessor_spec(prim["indices"])
        if spec.get("componentType") not in INDEX_COMPONENTS or spec.get("type") != "SCALAR":
            raise SceneError(f"{where}: indices must be a scalar u8/u16/u32 accessor")
        indices = reader.locate(prim["indices"])
        values = indices.array().ravel()
        n_indices = values.size
    else:
        n_indices = positions.count
    if n_indices % 3 != 0:
        raise SceneError(f"{where}: index count {n_indices} is not a multiple of 3")
    if values is not None and values.size and (values.min() < 0 or
                                               values.max() >= positions.count):
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
    return GltfPrimitiveRef(positions, normals, indices, n_indices, name, fallback), values


def _primitive(reader: _GltfReader, prim: dict, where: str, materials: list) -> GltfPrimitive:
    ref, values = _primitive_ref(reader, prim, where, materials)
    positions = ref.positions.array().astype(np.float64)
    normals = ref.normals.array().astype(np.float64) if ref.normals is not None else None
    indices = values.astype(np.int64) if values is not None else \
        np.arange(positions.shape[0], dtype=np.int64)
    return GltfPrimitive(positions, normals, indices, ref.material_name, ref.material_fallback)


def _primitive_located(reader, prim, where, materials) -> GltfPrimitiveRef:
    return _primitive_ref(reader, prim, where, materials)[0]


def load_gltf(path) -> GltfDocument:
    """Mesh-space geometry plus the node hierarchy of a .gltf / .glb file
    (scene.py:384-490)."""
    return _read_document(path, _primitive)


def load_gltf_located(path) -> GltfDocument:
    """load_gltf with every primitive left as located accessors
    (GltfPrimitiveRef): the same checks and errors, no float64 arrays."""
    return _read_document(path, _primitive_located)


def _read_document(path, primitive) -> GltfDocument:
    path = Path(path)
    if not path.is_file():
        raise SceneError(f"scene file not found: {path}")
    reader = _GltfReader(path)
    doc = reader.doc
    materials = doc.get("materials", [])
    meshes = []
    for mi, mesh in enumerate(doc.get("meshes", [])):
        name = mesh.get("name", f"mesh_{mi}")
        prims = [primitive(reader, prim, f"mesh {mi} ({name!r}) primitive {pi}", materials)
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


def _instances(doc: GltfDocument):
    """(world, linear, to_normals, primitive) per mesh primitive of every node
    in flatten_scene's depth-first visit order, with its cycle / singular
    transform checks (scene.py:527-560)."""
    def walk(idx: int, parent: np.ndarray, path: tuple):
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
                yield world, linear, to_normals, prim
        for child in node.children:
            yield from walk(child, world, path + (idx,))

    for root in doc.roots:
        yield from walk(root, np.eye(4), ())


class _MaterialSlots:
    """Material resolution (config name -> glTF fallback -> default) and the
    first-use slot table of flatten_scene."""

    def __init__(self, materials: MaterialMap):
        self.materials = materials
        self.table: dict = {}
        self.params_list: list = []

    def slot(self, prim) -> int:
        params = self.materials.resolve(prim.material_name) if prim.material_name else None
        if params is None:
            params = prim.material_fallback
        if params is None:
            params = self.materials.default
        if params not in self.table:
            self.table[params] = len(self.params_list)
            self.params_list.append(params)
        return self.table[params]


def flatten_scene(doc: GltfDocument, materials: MaterialMap, camera: CameraConfig,
                  environment: EnvironmentConfig) -> SceneDescription:
    """World-space triangle soup: node transforms baked in, materials
    resolved (config name -> glTF fallback -> default), degenerate triangles
    dropped (scene.py:519-596)."""
    parts = []
    slots = _MaterialSlots(materials)
    for world, linear, to_normals, prim in _instances(doc):
        world_pos = prim.positions @ linear.T + world[:3, 3]
        local_n = prim.normals if prim.normals is not None else \
            generate_smooth_normals(prim.positions, prim.indices)
        world_n = local_n @ to_normals.T
        slot = slots.slot(prim)
        ix = prim.indices
        parts.append(tuple(world_pos[ix[k::3]] for k in range(3)) +
                     tuple(world_n[ix[k::3]] for k in range(3)) + (slot,))
    params_list = slots.params_list
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


# ------------------------------------------------------------ device ingest

@contextlib.contextmanager
def _scene_errors():
    """The device flatten's all-degenerate verdict as the reference's
    SceneError("empty scene") (scene.py:582)."""
    try:
        yield
    except ValueError as exc:
        if str(exc) == "empty scene":
            raise SceneError("empty scene") from None
        raise


def gltf_device_desc(doc: GltfDocument, materials: MaterialMap):
    """The lt_gltf_desc of a located document (load_gltf_located): the
    buffers' raw bytes, one record per primitive, one per (node, primitive)
    instance in flatten_scene's visit order with its world matrix,
    inverse-transpose (computed here with the reference's numpy calls) and
    material slot.  Returns (desc, keep-alive list, material list, total
    triangles); raises the reference's "empty scene" for a scene with no
    triangles."""
    import ctypes as C

    from . import _lib
    keep: list = []
    buffers: list = []
    buffer_ids: dict = {}

    def buffer_of(loc: _Located) -> tuple[int, int, int]:
        if loc.data is None:        # an accessor without a bufferView: zeros
            data, first, stride = bytes(loc.count * loc.width * loc.dtype.itemsize), 0, \
                loc.width * loc.dtype.itemsize
        else:
            data, first, stride = loc.data, loc.first, loc.stride
        key = id(data)
        if key not in buffer_ids:
            buffer_ids[key] = len(buffers)
            buffers.append(data)
        return buffer_ids[key], first, stride

    prim_ids: dict = {}
    prims: list = []

    def prim_record(prim: GltfPrimitiveRef) -> int:
        key = id(prim)
        if key in prim_ids:
            return prim_ids[key]
        r = _lib.GltfPrimitive()
        r.pos_buffer, r.pos_offset, r.pos_stride = buffer_of(prim.positions)
        r.n_vertices = prim.positions.count
        if prim.normals is not None:
            r.nrm_buffer, r.nrm_offset, r.nrm_stride = buffer_of(prim.normals)
        else:
            r.nrm_buffer, r.nrm_offset, r.nrm_stride = -1, 0, 12
        if prim.indices is not None:
            r.idx_buffer, r.idx_offset, r.idx_stride = buffer_of(prim.indices)
            r.idx_bytes = prim.indices.dtype.itemsize
        else:
            r.idx_buffer, r.idx_offset, r.idx_stride, r.idx_bytes = -1, 0, 4, 4
        r.n_indices = prim.n_indices
        prim_ids[key] = len(prims)
        prims.append(r)
        keep.append(prim)
        return prim_ids[key]

    slots = _MaterialSlots(materials)
    instances = []
    total = 0
    for world, linear, to_normals, prim in _instances(doc):
        rec = _lib.GltfInstance()
        rec.primitive = prim_record(prim)
        rec.material = slots.slot(prim)
        rec.linear[:] = [float(x) for x in np.ascontiguousarray(linear).ravel()]
        rec.translation[:] = [float(x) for x in world[:3, 3]]
        rec.normal_matrix[:] = [float(x) for x in np.ascontiguousarray(to_normals).ravel()]
        instances.append(rec)
        total += prim.n_indices // 3
    if not instances or total == 0:
        raise SceneError("empty scene")
    desc = _lib.GltfDesc()
    desc.n_buffers = len(buffers)
    bufs = [np.frombuffer(b, dtype=np.uint8) if len(b) else np.zeros(1, np.uint8)
            for b in buffers]
    ptrs = (C.POINTER(C.c_uint8) * max(1, len(bufs)))(
        *[b.ctypes.data_as(C.POINTER(C.c_uint8)) for b in bufs])
    sizes = np.array([len(b) for b in buffers], dtype=np.int64)
    prim_arr = (_lib.GltfPrimitive * len(prims))(*prims)
    inst_arr = (_lib.GltfInstance * len(instances))(*instances)
    desc.buffers = ptrs
    desc.buffer_bytes = sizes.ctypes.data_as(C.POINTER(C.c_int64))
    desc.n_primitives = len(prims)
    desc.primitives = prim_arr
    desc.n_instances = len(instances)
    desc.instances = inst_arr
    keep += [buffers, bufs, ptrs, sizes, prim_arr, inst_arr]
    return desc, keep, slots.params_list, total


def flatten_scene_device(doc: GltfDocument, materials: MaterialMap, camera: CameraConfig,
                         environment: EnvironmentConfig, device: int = 0) -> SceneDescription:
    """flatten_scene (scene.py:519-596) on the GPU from a located document:
    the same SceneDescription bit for bit (lt_gltf_flatten), copied back to
    the host."""
    import ctypes as C

    from . import _lib
    _lib.require_gpu()
    desc, keep, params_list, total = gltf_device_desc(doc, materials)
    out = [np.empty((total, 3)) for _ in range(6)]
    mat = np.empty(total, dtype=np.int32)
    kept, dropped = C.c_int64(0), C.c_int64(0)
    dp = C.POINTER(C.c_double)
    with _scene_errors():
        _lib.check(_lib.lib().lt_gltf_flatten(
            C.byref(desc), int(device), total, *[a.ctypes.data_as(dp) for a in out],
            mat.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(kept), C.byref(dropped)))
    k = kept.value
    tris = TriangleBuffer(*[a[:k] for a in out], mat[:k])
    return SceneDescription(tris, params_list, camera, environment, dropped.value)


def load_scene_gpu(scene_path, config_path, device: int = 0) -> SceneDescription:
    """load_scene with the flatten on the GPU: the host reads the file and
    walks the nodes, the device decodes the float32 accessors and builds the
    world-space soup; the result is load_scene's, bit for bit."""
    config = load_render_config(config_path)
    return flatten_scene_device(load_gltf_located(scene_path), config.materials, config.camera,
                                config.environment, device)


def load_device_scene(scene_path, config_path, device: int = 0):
    """glTF file + render config straight to a resident DeviceScene: the
    GLB's float32 / integer bytes are the only geometry uploaded, the
    flattened soup and the BVH are built on the device
    (lt_scene_create_gltf).  `render_progressive(ds, settings)` renders it;
    `ds.degenerate_dropped` and `ds.camera` are set."""
    from .device import DeviceScene
    config = load_render_config(config_path)
    doc = load_gltf_located(scene_path)
    desc, keep, params_list, _ = gltf_device_desc(doc, config.materials)
    with _scene_errors():
        ds = DeviceScene.from_gltf(desc, keep, params_list, config.environment, config.camera,
                                   device)
    ds.materials = params_list
    return ds


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

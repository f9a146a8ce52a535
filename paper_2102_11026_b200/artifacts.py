"""Artifact I/O of the trained models the hot path consumes.

Formats follow the reference SPEC's External Interfaces:
  * densenet checkpoint: JSON with layer specs, row-major weight arrays, seed and
    training metadata; bit-exact round trip (floats are written with Python's shortest
    round-tripping repr);
  * PoseSet: binary header (N, T) as two little-endian int64, then the N x T
    poses column-major (pose after pose) as float64, then the T energies; plus a JSON sidecar
    ``<path>.json`` with the generating script;
  * ReducedModel: U in the PoseSet format + decoder / encoder checkpoints + a JSON
    manifest;
  * CubatureModel: element-id list + weight-net / selection-net checkpoints +
    manifest;
  * mesh: plain text, header line "N_vertices N_tets", the coordinates, the 4-index
    tets, then optionally a line "N_triangles" and the surface triangles.
Host-side only: loading produces the same numpy arrays the GPU session uploads.
"""

from __future__ import annotations

import json
import os

import numpy as np

from .densenet import DenseNet

_I64 = np.dtype("<i8")
_F64 = np.dtype("<f8")


# ----------------------------------------------------------------------------- densenet
def save_checkpoint(net: DenseNet, path: str, metadata: dict | None = None) -> None:
    doc = json.loads(net.to_json())
    doc["metadata"] = dict(metadata or {})
    with open(path, "w") as f:
        json.dump(doc, f)


def load_checkpoint(path: str) -> DenseNet:
    with open(path) as f:
        doc = json.load(f)
    net = DenseNet.from_json(json.dumps({k: v for k, v in doc.items() if k != "metadata"}))
    net.metadata = doc.get("metadata", {})
    return net


# ----------------------------------------------------------------------------- PoseSet
def save_poseset(path: str, poses, energies=None, script: dict | None = None) -> None:
    """poses: (N, T) -- one column per pose."""
    X = np.asarray(poses, dtype=float)
    if X.ndim != 2:
        raise ValueError("dimension mismatch: poses must be (N, T)")
    N, T = X.shape
    e = np.zeros(T) if energies is None else np.asarray(energies, dtype=float).reshape(-1)
    if e.size != T:
        raise ValueError("dimension mismatch: one energy per pose")
    with open(path, "wb") as f:
        f.write(np.array([N, T], dtype=_I64).tobytes())
        f.write(np.asfortranarray(X).astype(_F64).tobytes(order="F"))
        f.write(e.astype(_F64).tobytes())
    with open(path + ".json", "w") as f:
        json.dump({"script": script or {}, "N": int(N), "T": int(T)}, f)


def load_poseset(path: str):
    """-> (poses (N, T), energies (T,), script dict)."""
    with open(path, "rb") as f:
        raw = f.read()
    N, T = (int(v) for v in np.frombuffer(raw[:16], dtype=_I64))
    if len(raw) != 16 + 8 * (N * T + T):
        raise ValueError("PoseSet file size does not match its header")
    X = np.frombuffer(raw[16:16 + 8 * N * T], dtype=_F64).reshape((N, T), order="F").copy()
    e = np.frombuffer(raw[16 + 8 * N * T:], dtype=_F64).copy()
    script = {}
    if os.path.exists(path + ".json"):
        with open(path + ".json") as f:
            script = json.load(f).get("script", {})
    return X, e, script


# ----------------------------------------------------------------------------- ReducedModel
def save_reduced_model(rm, directory: str) -> None:
    os.makedirs(directory, exist_ok=True)
    save_poseset(os.path.join(directory, "U.poseset"), rm.U)
    save_checkpoint(rm.decoder, os.path.join(directory, "decoder.json"))
    files = {"U": "U.poseset", "decoder": "decoder.json"}
    if rm.encoder is not None:
        save_checkpoint(rm.encoder, os.path.join(directory, "encoder.json"))
        files["encoder"] = "encoder.json"
    with open(os.path.join(directory, "manifest.json"), "w") as f:
        json.dump({"kind": "ReducedModel", "n_p": rm.n_p, "n_q": rm.n_q, "N": int(rm.U.shape[0]), "files": files}, f)


def load_reduced_model(directory: str):
    from .daereduce import ReducedModel
    with open(os.path.join(directory, "manifest.json")) as f:
        man = json.load(f)
    if man.get("kind") != "ReducedModel":
        raise ValueError("not a ReducedModel manifest")
    U, _, _ = load_poseset(os.path.join(directory, man["files"]["U"]))
    dec = load_checkpoint(os.path.join(directory, man["files"]["decoder"]))
    enc = None
    if "encoder" in man["files"]:
        enc = load_checkpoint(os.path.join(directory, man["files"]["encoder"]))
    if U.shape != (man["N"], man["n_p"]):
        raise ValueError("dimension mismatch between the manifest and U")
    return ReducedModel(U, dec, man["n_p"], man["n_q"], encoder=enc)


# ----------------------------------------------------------------------------- CubatureModel
def save_cubature_model(cm, directory: str) -> None:
    os.makedirs(directory, exist_ok=True)
    files = {}
    if cm.wnet is not None:
        save_checkpoint(cm.wnet, os.path.join(directory, "wnet.json"))
        files["wnet"] = "wnet.json"
    if isinstance(cm.snet, DenseNet):
        save_checkpoint(cm.snet, os.path.join(directory, "snet.json"))
        files["snet"] = "snet.json"
    with open(os.path.join(directory, "manifest.json"), "w") as f:
        json.dump({"kind": "CubatureModel", "C": [int(e) for e in cm.C], "K": int(cm.K), "files": files}, f)


def load_cubature_model(directory: str):
    from .neucubature import CubatureModel
    with open(os.path.join(directory, "manifest.json")) as f:
        man = json.load(f)
    if man.get("kind") != "CubatureModel":
        raise ValueError("not a CubatureModel manifest")
    wnet = load_checkpoint(os.path.join(directory, man["files"]["wnet"])) if "wnet" in man["files"] else None
    snet = load_checkpoint(os.path.join(directory, man["files"]["snet"])) if "snet" in man["files"] else None
    return CubatureModel(np.asarray(man["C"], dtype=np.int32), wnet, snet, man.get("K", 5))


# ----------------------------------------------------------------------------- mesh
def write_mesh(mesh, path: str) -> None:
    with open(path, "w") as f:
        f.write(f"{mesh.vertices.shape[0]} {mesh.tets.shape[0]}\n")
        for v in mesh.vertices:
            f.write(" ".join(repr(float(x)) for x in v) + "\n")
        for t in mesh.tets:
            f.write(" ".join(str(int(i)) for i in t) + "\n")
        if mesh.surface is not None and len(mesh.surface):
            f.write(f"{len(mesh.surface)}\n")
            for t in mesh.surface:
                f.write(" ".join(str(int(i)) for i in t) + "\n")


def read_mesh(path: str):
    from .elastic import TetMesh
    with open(path) as f:
        lines = [ln.split() for ln in f if ln.strip()]
    V, T = int(lines[0][0]), int(lines[0][1])
    verts = np.array([[float(x) for x in ln] for ln in lines[1:1 + V]], dtype=float)
    tets = np.array([[int(x) for x in ln] for ln in lines[1 + V:1 + V + T]], dtype=np.int32)
    if verts.shape != (V, 3) or tets.shape != (T, 4):
        raise ValueError("mesh file does not match its header")
    surface = None
    rest = lines[1 + V + T:]
    if rest:
        S = int(rest[0][0])
        surface = np.array([[int(x) for x in ln] for ln in rest[1:1 + S]], dtype=np.int32)
        if surface.shape != (S, 3):
            raise ValueError("surface triangle block does not match its count")
    return TetMesh(verts, tets, surface)

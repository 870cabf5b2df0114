"""PSHARD01 checkpoints — byte-compatible with phantomsim.checkpoint (reference checkpoint.py:1-110).

Layout (little endian), as the reference writes it:

    magic "PSHARD01" | mode u8 (0 phantom, 1 tensor) | n, p, k, layers, seed  i64 each
    | one activation code u8 per layer (0 relu, 1 identity)
    | float64 row-major matrices: for each rank, for each layer
          phantom: local [s,s], compressor [k,s], decompressors [s,k] ascending source rank
                   (self excluded), bias [s]
          tensor:  weight [s,n], bias [s]

The file layout is fixed by (mode, n, p, k, layers), so every (rank, layer) block has a known
byte offset: a multi-GPU engine writes and reads only its own logical ranks' blocks in place
(no gather to one process).  Values go through the fp32 master (f64 -> fp32 -> f64), so a
checkpoint whose values are fp32-representable round-trips byte for byte.

Resume (which the reference lacks): `save_state` writes the PSHARD01 weights plus a sidecar
`<path>.ppxopt` with the optimizer state (step count, Adam moments in the same block order).
"""

from __future__ import annotations

import os
import struct
from pathlib import Path

import numpy as np
import torch

from .core import Activation, as_activation
from .errors import ConfigurationError

MAGIC = b"PSHARD01"
_HEADER = struct.Struct("<8sBqqqqq")
_ACT_CODE = {Activation.RELU: 0, Activation.IDENTITY: 1}
_ACT_FROM = {code: act for act, code in _ACT_CODE.items()}
OPT_MAGIC = b"PPXOPT01"
_OPT_HEADER = struct.Struct("<8sBqq")   # magic, kind (0 sgd, 1 adam), step t, f64 count per moment


# ----------------------------------------------------------------------------------------------
# format geometry (host only: shared by the device models, the engine and the CPU tests)
# ----------------------------------------------------------------------------------------------
class Geometry:
    """Byte offsets of every block of a PSHARD01 file (checkpoint.py:57-64 order)."""

    def __init__(self, mode: int, n: int, p: int, k: int, layers: int):
        if mode not in (0, 1):
            raise ConfigurationError(f"unknown mode byte {mode}")
        if p < 1 or n % p:
            raise ConfigurationError(f"n={n} not divisible by p={p}")
        self.mode, self.n, self.p, self.k, self.layers = mode, n, p, k, layers
        self.s = s = n // p
        if mode == 0:
            self.shapes = [("local", (s, s)), ("compressor", (k, s))] + \
                          [("dec", (s, k))] * (p - 1) + [("bias", (s,))]
        else:
            self.shapes = [("weight", (s, n)), ("bias", (s,))]
        self.block_elems = sum(int(np.prod(sh)) for _, sh in self.shapes)
        self.data_start = _HEADER.size + layers

    def block_offset(self, rank: int, layer: int) -> int:
        return self.data_start + 8 * self.block_elems * (rank * self.layers + layer)

    @property
    def file_size(self) -> int:
        return self.data_start + 8 * self.block_elems * self.p * self.layers


def _header_bytes(mode, n, p, k, layers, seed, activations) -> bytes:
    return _HEADER.pack(MAGIC, mode, n, p, k, layers, seed) + bytes(_ACT_CODE[as_activation(a)] for a in activations)


def read_header(path):
    """(mode, n, p, k, layers, seed, activations) with the reference's validation
    (checkpoint.py:72-88)."""
    path = Path(path)
    with open(path, "rb") as fh:
        header = fh.read(_HEADER.size)
        if len(header) != _HEADER.size:
            raise ConfigurationError(f"{path}: not a checkpoint (short header)")
        magic, mode, n, p, k, layers, seed = _HEADER.unpack(header)
        if magic != MAGIC:
            raise ConfigurationError(f"{path}: bad magic {magic!r}")
        if mode not in (0, 1):
            raise ConfigurationError(f"{path}: unknown mode byte {mode}")
        act_bytes = fh.read(layers)
        if len(act_bytes) != layers:
            raise ConfigurationError(f"{path}: truncated activation table")
        try:
            acts = [_ACT_FROM[b] for b in act_bytes]
        except KeyError as exc:
            raise ConfigurationError(f"{path}: unknown activation code {exc}") from None
    return mode, n, p, k, layers, seed, acts


def _block_arrays(raw: bytes, geo: Geometry) -> list:
    vals = np.frombuffer(raw, dtype="<f8")
    out, pos = [], 0
    for _, sh in geo.shapes:
        cnt = int(np.prod(sh))
        out.append(vals[pos:pos + cnt].reshape(sh).astype(np.float64))
        pos += cnt
    return out


def read_block(path, geo: Geometry, rank: int, layer: int) -> list:
    """The float64 matrices of one (rank, layer) block, in file order."""
    with open(path, "rb") as fh:
        fh.seek(geo.block_offset(rank, layer))
        raw = fh.read(8 * geo.block_elems)
    if len(raw) != 8 * geo.block_elems:
        raise ConfigurationError(f"{path}: checkpoint truncated")
    return _block_arrays(raw, geo)


def check_size(path, geo: Geometry) -> None:
    size = os.path.getsize(path)
    if size < geo.file_size:
        raise ConfigurationError(f"{path}: checkpoint truncated")
    if size > geo.file_size:
        raise ConfigurationError(f"{path}: trailing bytes after matrices")


def _block_bytes(mats) -> bytes:
    return b"".join(np.ascontiguousarray(np.asarray(m, dtype=np.float64), dtype="<f8").tobytes() for m in mats)


def _to_host(t) -> np.ndarray:
    if isinstance(t, torch.Tensor):
        return t.detach().to(torch.float64).cpu().numpy()
    return np.asarray(t, dtype=np.float64)


def write_block(fh, geo: Geometry, rank: int, layer: int, mats) -> None:
    data = _block_bytes(mats)
    if len(data) != 8 * geo.block_elems:
        raise ConfigurationError("block does not match the checkpoint geometry")
    fh.seek(geo.block_offset(rank, layer))
    fh.write(data)


# ----------------------------------------------------------------------------------------------
# reference-API models (phantom.PhantomModel / tensor_parallel.TPModel)
# ----------------------------------------------------------------------------------------------
def _phantom_mats(layer, rank, p):
    if isinstance(layer, dict):
        get = layer.__getitem__
    else:
        get = lambda nm: getattr(layer, nm)   # noqa: E731
    decs = get("decompressors")
    return [_to_host(get("local")), _to_host(get("compressor"))] + \
           [_to_host(decs[i]) for i in sorted(decs)] + [_to_host(get("bias"))]


def save_model(path, model) -> None:
    """checkpoint.py:44-62 — write a phantom or tensor model (device tensors are read back)."""
    from .phantom import PhantomModel
    from .tensor_parallel import TPModel
    is_pp = isinstance(model, PhantomModel)
    if not is_pp and not isinstance(model, TPModel):
        raise ConfigurationError(f"cannot checkpoint a {type(model).__name__}")
    k = model.k if is_pp else 0
    geo = Geometry(0 if is_pp else 1, model.n, model.p, k, model.layer_count)
    with open(Path(path), "wb") as fh:
        fh.write(_header_bytes(geo.mode, model.n, model.p, k, model.layer_count, model.seed, model.activations))
        for rank in range(model.p):
            row = model.rank_layers[rank]
            if row is None:
                raise ConfigurationError(f"rank {rank} is not materialised in this process")
            for l, layer in enumerate(row):
                mats = _phantom_mats(layer, rank, model.p) if is_pp else [_to_host(layer.weight), _to_host(layer.bias)]
                write_block(fh, geo, rank, l, mats)


def load_model(path, *, dtype=None, device=None):
    """checkpoint.py:65-110 — read a checkpoint into a device PhantomModel / TPModel."""
    from .phantom import DEFAULT_DTYPE, PhantomLayer, PhantomModel
    from .tensor_parallel import TPLayer, TPModel
    mode, n, p, k, layers, seed, acts = read_header(path)
    geo = Geometry(mode, n, p, k, layers)
    check_size(path, geo)
    dev = torch.device(device or "cuda")
    rank_layers = []
    for rank in range(p):
        own = []
        for l in range(layers):
            mats = read_block(path, geo, rank, l)
            if mode == 0:
                decs = {i: mats[2 + q] for q, i in enumerate(i for i in range(p) if i != rank)}
                own.append(PhantomLayer(mats[0], mats[1], decs, mats[-1], rank=rank, p=p,
                                        dtype=dtype or DEFAULT_DTYPE, device=dev))
            else:
                own.append(TPLayer(torch.from_numpy(mats[0]).to(dev, dtype or torch.float32),
                                   torch.from_numpy(mats[1]).to(dev, dtype or torch.float32)))
        rank_layers.append(own)
    if mode == 0:
        return PhantomModel(n, p, k, acts, rank_layers, seed)
    return TPModel(n, p, acts, rank_layers, seed)


# ----------------------------------------------------------------------------------------------
# the training engine (engine.PhantomEngine): each process handles only its logical ranks
# ----------------------------------------------------------------------------------------------
def _engine_geometry(eng) -> Geometry:
    return Geometry(0, eng.n, eng.p, eng.k, eng.L)


def save_engine(path, eng, seed: int = 0, *, create: bool = True, barrier=None) -> None:
    """Write the engine's fp32 master weights as PSHARD01.  With several processes, `create` is
    True on the process that writes the header and sizes the file (call `barrier` between) and
    every process writes its own ranks' blocks in place."""
    geo = _engine_geometry(eng)
    path = Path(path)
    if create:
        with open(path, "wb") as fh:
            fh.write(_header_bytes(0, eng.n, eng.p, eng.k, eng.L, seed, [eng.act] * eng.L))
            fh.truncate(geo.file_size)
    if barrier is not None:
        barrier()
    torch.cuda.synchronize()
    with open(path, "r+b") as fh:
        for jj, j in enumerate(eng.local):
            for l in range(eng.L):
                write_block(fh, geo, j, l, _phantom_mats(eng.layer_views(jj, l), j, eng.p))
    if barrier is not None:
        barrier()


def load_engine(path, eng) -> int:
    """Load this process's logical ranks from a PSHARD01 file into the engine (weights and the
    compute copies); returns the checkpoint's seed."""
    mode, n, p, k, layers, seed, acts = read_header(path)
    if mode != 0 or (n, p, k, layers) != (eng.n, eng.p, eng.k, eng.L):
        raise ConfigurationError(f"{path}: checkpoint (mode {mode}, n={n}, p={p}, k={k}, L={layers}) does not "
                                 f"match the engine (n={eng.n}, p={eng.p}, k={eng.k}, L={eng.L})")
    geo = Geometry(mode, n, p, k, layers)
    check_size(path, geo)
    rows = {}
    for j in eng.local:
        row = []
        for l in range(layers):
            mats = read_block(path, geo, j, l)
            decs = {i: mats[2 + q] for q, i in enumerate(i for i in range(p) if i != j)}
            row.append({"local": mats[0], "compressor": mats[1], "decompressors": decs, "bias": mats[-1]})
        rows[j] = row
    eng.load_params(rows)
    return seed


def save_state(path, eng, seed: int = 0, *, create: bool = True, barrier=None) -> None:
    """Weights (PSHARD01) plus the optimizer state sidecar <path>.ppxopt for an exact resume."""
    save_engine(path, eng, seed, create=create, barrier=barrier)
    geo = _engine_geometry(eng)
    adam = eng.optimizer == "adam"
    side = Path(str(path) + ".ppxopt")
    per_moment = geo.block_elems * geo.p * geo.layers
    if create:
        with open(side, "wb") as fh:
            fh.write(_OPT_HEADER.pack(OPT_MAGIC, 1 if adam else 0, int(eng.t), per_moment if adam else 0))
            if adam:
                fh.truncate(_OPT_HEADER.size + 2 * 8 * per_moment)
    if barrier is not None:
        barrier()
    if adam:
        torch.cuda.synchronize()
        with open(side, "r+b") as fh:
            for which, (mom, bmom) in enumerate(((eng.adam_m, eng.adam_bm), (eng.adam_v, eng.adam_bv))):
                for jj, j in enumerate(eng.local):
                    for l in range(eng.L):
                        v = eng.layer_views(jj, l, master=mom[jj, l], bias=bmom[jj, l])
                        data = _block_bytes(_phantom_mats(v, j, eng.p))
                        fh.seek(_OPT_HEADER.size + 8 * per_moment * which + (geo.block_offset(j, l) - geo.data_start))
                        fh.write(data)
    if barrier is not None:
        barrier()


def load_state(path, eng) -> int:
    """Inverse of save_state: weights, step count and (Adam) moments; returns the seed."""
    seed = load_engine(path, eng)
    side = Path(str(path) + ".ppxopt")
    if not side.exists():
        raise ConfigurationError(f"{side}: optimizer state missing (use load_engine for weights only)")
    geo = _engine_geometry(eng)
    with open(side, "rb") as fh:
        head = fh.read(_OPT_HEADER.size)
        if len(head) != _OPT_HEADER.size:
            raise ConfigurationError(f"{side}: short header")
        magic, kind, t, per_moment = _OPT_HEADER.unpack(head)
        if magic != OPT_MAGIC:
            raise ConfigurationError(f"{side}: bad magic {magic!r}")
        if (kind == 1) != (eng.optimizer == "adam"):
            raise ConfigurationError(f"{side}: optimizer kind does not match the engine")
        eng.set_step_count(int(t))
        if kind == 1:
            if per_moment != geo.block_elems * geo.p * geo.layers:
                raise ConfigurationError(f"{side}: moment size does not match the engine")
            for which, (mom, bmom) in enumerate(((eng.adam_m, eng.adam_bm), (eng.adam_v, eng.adam_bv))):
                for jj, j in enumerate(eng.local):
                    for l in range(eng.L):
                        fh.seek(_OPT_HEADER.size + 8 * per_moment * which + (geo.block_offset(j, l) - geo.data_start))
                        raw = fh.read(8 * geo.block_elems)
                        if len(raw) != 8 * geo.block_elems:
                            raise ConfigurationError(f"{side}: truncated")
                        mats = _block_arrays(raw, geo)
                        v = eng.layer_views(jj, l, master=mom[jj, l], bias=bmom[jj, l])
                        v["local"].copy_(torch.from_numpy(mats[0]))
                        v["compressor"].copy_(torch.from_numpy(mats[1]))
                        for q, i in enumerate(i for i in range(eng.p) if i != j):
                            v["decompressors"][i].copy_(torch.from_numpy(mats[2 + q]))
                        v["bias"].copy_(torch.from_numpy(mats[-1]))
    return seed

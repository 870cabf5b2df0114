"""PhantomEngine — the throughput path: one process per GPU, NCCL over NVLink, CUDA graphs.

The engine runs `pp_iteration` + the optimizer (reference training.py:181-213, 276-309) for the
logical ranks this GPU owns, natively in [batch, features] layout, with every dense contraction
in the tcgen05 kernel and these fusions:

  forward  layer l:  compress (K2) -> phantom all-gather on the comm stream -> ONE
                     K-concatenated local+decompress GEMM with bias+ReLU epilogue (K1); the
                     output layer's epilogue also forms delta_L, the loss partial and d bias (K7/K8).
  backward layer l:  error compression D^T delta (K3) -> reduce-scatter on the comm stream,
                     overlapped with the grouped weight-gradient launch {d local_l, d decomp_l,
                     d compressor_{l+1}} whose epilogue applies SGD/Adam in place (K4/K5/K9);
                     then [delta | r].[L ; C] with the ReLU'-mask + d bias epilogue (K6/K8).

Logical rank j lives on GPU j // R (R = p / world).  Weights are fp32 masters plus two bf16
compute copies (read one, write the other: the update of step t never races the GEMMs of step
t that still read the old weights).  Each step is captured once per parity in a CUDA graph.
"""

from __future__ import annotations

import ctypes
import math
import os

import torch

from . import _lib, kernels
from .core import Activation, as_activation, flat_offsets, round8
from .errors import ConfigurationError, TrainingError
from .schedule import local_ranks


def pp_step_flops(n: int, p: int, k: int, layers: int, batch: int) -> int:
    """Algorithmic GEMM FLOPs of one training step for ONE logical rank:
    6 L B s (s + p k) - 2 B s (s + k)  (layer 0 has no error recurrence)."""
    s = n // p
    return 6 * layers * batch * s * (s + p * k) - 2 * batch * s * (s + k)


def pp_forward_flops(n: int, p: int, k: int, layers: int, batch: int) -> int:
    s = n // p
    return 2 * layers * batch * s * (s + p * k)


def _dist_barrier():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.barrier()


class PhantomEngine:
    def __init__(self, n: int, p: int, k: int, layers: int, batch: int, *, world: int = 1, rank: int = 0,
                 device: int = 0, uid: bytes | None = None, activation=Activation.RELU, reduction: str = "mean",
                 optimizer: str = "sgd", lr: float = 1e-4, betas=(0.9, 0.999), eps: float = 1e-8,
                 dtype: torch.dtype = torch.bfloat16, seed: int = 0, ctx: _lib.Context | None = None):
        if n % p:
            raise ConfigurationError(f"n={n} not divisible by p={p}")
        if p % world:
            raise ConfigurationError(f"p={p} logical ranks do not divide over {world} GPUs")
        s = n // p
        if not 1 <= k <= s:
            raise ConfigurationError(f"need 1 <= k <= n/p, got k={k}, n/p={s}")
        if optimizer not in ("sgd", "adam"):
            raise ConfigurationError("optimizer must be sgd or adam")
        self.n, self.p, self.k, self.L, self.B, self.s = n, p, k, layers, batch, s
        self.world, self.rank, self.R = world, rank, p // world
        self.local = local_ranks(p, world, rank)
        self.act = as_activation(activation)
        self.reduction, self.optimizer, self.lr, self.betas, self.eps = reduction, optimizer, lr, betas, eps
        self.dtype = dtype
        self.pdt = kernels.ppx_dtype(dtype)
        self.dev = torch.device("cuda", device)
        torch.cuda.set_device(self.dev)
        self.ctx = ctx or _lib.Context(world, rank, device, uid)
        self.comm_stream = torch.cuda.Stream(self.dev)
        self.copy_stream = torch.cuda.Stream(self.dev)
        self.off = flat_offsets(s, k, p)
        T, R, L, B = self.off["total"], self.R, layers, batch
        ldk = self.off["ldk"]
        f32 = torch.float32
        # parameters
        self.master = torch.zeros((R, L, T), dtype=f32, device=self.dev)
        # two compute copies (read w[par], the fused update writes w[1-par]); separate from the
        # master even in the fp32 tier so an in-place update never races a GEMM of the same step
        self.w = [torch.zeros((R, L, T), dtype=dtype, device=self.dev) for _ in range(2)]
        self.bias = torch.zeros((R, L, s), dtype=f32, device=self.dev)
        self.gbias = torch.zeros((R, L, s), dtype=f32, device=self.dev)
        if optimizer == "adam":
            self.adam_m = torch.zeros_like(self.master)
            self.adam_v = torch.zeros_like(self.master)
            self.adam_bm = torch.zeros_like(self.bias)
            self.adam_bv = torch.zeros_like(self.bias)
        self.t = 0
        self._init_weights(seed)
        # activations: Y[parity][jj][l], l = 0 (input) .. L (output); targets per parity
        self.Y = [[[torch.empty((B, s), dtype=dtype, device=self.dev) for _ in range(L + 1)] for _ in range(R)]
                  for _ in range(2)]
        # the inner layers' activations are shared between parities (only inputs double-buffer)
        for jj in range(R):
            for l in range(1, L + 1):
                self.Y[1][jj][l] = self.Y[0][jj][l]
        self.Tgt = [[torch.empty((B, s), dtype=dtype, device=self.dev) for _ in range(R)] for _ in range(2)]
        self.D = [[torch.empty((B, s), dtype=dtype, device=self.dev) for _ in range(2)] for _ in range(R)]
        # phantom all-gather buffers; on multi-GPU runs the batch is split in two halves
        # [2][p][B/2, ldk] so each half's all-gather hides behind the other half's GEMMs
        self.halves = 2 if (world > 1 and B % 128 == 0 and os.environ.get("PPX_HALVES", "1") == "2") else 1
        # NVLink phantom exchange (world > 1): the G buffers live in IPC-shared memory; the
        # compression GEMM stores every phantom tile into all peers' G buffers and a per-layer
        # flag replaces the NCCL all-gather (PPX_P2P=1; default NCCL)
        self.bad = torch.zeros(1, dtype=torch.int32, device=self.dev)
        # default (PPX_FUSED=0 disables; bf16, 64-aligned s and k): compression + all-gather + forward of a layer as ONE launch of the
        # 2-SM kernel — compression tiles store their phantoms into every GPU's buffer over
        # NVLink and bump per-layer arrival counters, forward tiles wait in-kernel after their
        # local-block segment
        self.fused = (os.environ.get("PPX_FUSED", "1") != "0" and dtype == torch.bfloat16 and s % 64 == 0
                      and k % 64 == 0 and p // world <= 8 and not os.environ.get("PPX_NOGROUP")
                      and (world == 1 or self._dist_ready()))
        self.p2p = int(os.environ.get("PPX_P2P", "0")) if world > 1 and self._dist_ready() else 0
        if self.fused and world > 1 and not self.p2p:
            self.p2p = 2
        if self.p2p:
            self.halves = 1
            self._setup_p2p(dtype)
        else:
            self.G = [torch.zeros((p, B, ldk), dtype=dtype, device=self.dev) for _ in range(L)]
        if self.fused:
            self.halves = 1
            self._setup_fused()
        self.H = [torch.zeros((p, B, ldk), dtype=dtype, device=self.dev) for _ in range(L)]
        # out-of-place reduce-scatter target (world > 1): this GPU's R received slots
        self.Hr = [torch.zeros((R, B, ldk), dtype=dtype, device=self.dev) for _ in range(L)] if world > 1 else None
        self.loss = torch.zeros(1, dtype=f32, device=self.dev)
        self.hyper = torch.zeros(6, dtype=f32, device=self.dev)
        self.hyper_host = torch.zeros(6, dtype=f32).pin_memory()
        self.out_host = torch.zeros(1, dtype=f32).pin_memory()
        self.bad_host = torch.zeros(1, dtype=torch.int32).pin_memory()
        if dtype == torch.float32:   # 3xTF32 hi/lo splits: reserve so graph capture never allocates
            per_call = 4 * B * s + 2 * p * B * ldk + 2 * T + 4 * s * ldk
            self.ctx.call("ppx_reserve_workspace", int(2 * 4 * per_call * 1.25) + (1 << 20))
        self.comm_sms = int(os.environ.get("PPX_COMM_SMS", "0"))
        # PPX_NOGROUP=1 launches every logical rank separately (emulates the R=1 launch shapes of an
        # 8-GPU run on one GPU, for profiling)
        self.group = 1 if os.environ.get("PPX_NOGROUP") else R
        self.graphs = [None, None]
        self.parity = 0
        # training steps skip the output layer's y store (PPX_STORE_OUTPUT=1 keeps it)
        self.skip_output = not os.environ.get("PPX_STORE_OUTPUT")
        # weight gradients + error recurrence of a layer as one LPT-scheduled launch (after the
        # reduce-scatter): default with one logical rank per GPU, where either launch alone leaves
        # ~1.4 rounds of tiles (PPX_BWD_FUSED=1/0 forces it on / off)
        bf = os.environ.get("PPX_BWD_FUSED", "")
        self.bwd_fused = dtype == torch.bfloat16 and (bf == "1" or (bf == "" and self.R == 1 and world > 1))
        # timing experiments ONLY (wrong results): drop the backward reduce-scatter
        self._dbg_skip_rs = bool(os.environ.get("PPX_DEBUG_SKIP_RS"))
        self._dbg_skip_ag = bool(os.environ.get("PPX_DEBUG_SKIP_AG"))
        self._keep = []   # ctypes structs of the launch being built
        self._launches = 0
        self.launch_count = 0
        self.trace = []   # kernel-launching ABI calls of the last step body (profiling labels)

    # ------------------------------------------------------------------------------------------
    @staticmethod
    def _dist_ready():
        import torch.distributed as dist
        return dist.is_available() and dist.is_initialized()

    def _setup_p2p(self, dtype):
        """IPC region [L][p, B, ldk] phantoms + [L][world] int32 flags on every GPU, mapped by all
        peers (handles exchanged over torch.distributed); identical layouts, so a peer address
        is peer_base + (local address - local base)."""
        import torch.distributed as dist
        p, B, L, ldk, world = self.p, self.B, self.L, self.off["ldk"], self.world
        esz = torch.tensor([], dtype=dtype).element_size()
        gbytes = p * B * ldk * esz
        self._goff = [l * gbytes for l in range(L)]
        self._foff = L * gbytes
        self._coff = self._foff + ((L * world * 4 + 255) // 256) * 256    # per-layer arrival counters
        self._rcoff = self._coff + ((L * 4 + 255) // 256) * 256           # reduce-scatter arrival counters
        sbytes = world * self.R * B * ldk * esz                           # reduce-scatter staging per layer
        self._soff = [self._rcoff + ((L * 4 + 255) // 256) * 256 + l * sbytes for l in range(L)]
        nbytes = self._soff[0] + L * sbytes
        ptr = ctypes.c_void_p()
        handle = ctypes.create_string_buffer(64)
        self.ctx.call("ppx_peer_alloc", nbytes, ctypes.byref(ptr), handle)
        self._pbase = ptr.value
        handles = [None] * world
        dist.all_gather_object(handles, handle.raw)
        self._peer_base = {}
        for g in range(world):
            if g != self.rank:
                q = ctypes.c_void_p()
                self.ctx.call("ppx_peer_open", handles[g], ctypes.byref(q))
                self._peer_base[g] = q.value
        self._peers = [g for g in range(world) if g != self.rank]

        class _Raw:   # torch view of the region (owned by the ctx, freed by ppx_destroy)
            def __init__(self, addr, n):
                self.__cuda_array_interface__ = {"shape": (n,), "typestr": "|u1", "data": (addr, False),
                                                 "version": 3}
        raw = torch.as_tensor(_Raw(self._pbase, nbytes), device=self.dev)
        self.G = [raw[o:o + gbytes].view(dtype).view(p, B, ldk) for o in self._goff]
        self._sigcnt = torch.zeros(L, dtype=torch.int32, device=self.dev)
        self._waitcnt = torch.zeros(L, dtype=torch.int32, device=self.dev)
        n = len(self._peers)
        mk = lambda addrs: (ctypes.c_void_p * max(n, 1))(*addrs)   # noqa: E731
        self._push_dst = [mk([self._peer_base[g] + o for g in self._peers]) for o in self._goff]
        # flag (l, src) lives at foff + 4 (l * world + src) in the region of the GPU that waits
        self._sig_dst = [mk([self._peer_base[g] + self._foff + 4 * (l * world + self.rank) for g in self._peers])
                         for l in range(L)]
        self._wait_src = [mk([self._pbase + self._foff + 4 * (l * world + g) for g in self._peers])
                          for l in range(L)]
        # NVLink reduce-scatter (bf16, with the IPC region): default when a GPU owns >= 2 logical
        # ranks (C3 on 4 GPUs: 5.41 -> 5.31 ms); with one rank per GPU the per-slot error
        # compression tiles worse than the NCCL path (C2 on 4 GPUs: 2.53 -> 2.70 ms), so it is
        # opt-in there (PPX_NVRS=1; PPX_NVRS=0 always NCCL)
        nv = os.environ.get("PPX_NVRS", "")
        self.nvrs = dtype == torch.bfloat16 and self.R <= 8 and (nv == "1" or (nv == "" and self.R >= 2))
        if self.nvrs:
            vpp = ctypes.POINTER(ctypes.c_void_p)
            base = lambda g: self._pbase if g == self.rank else self._peer_base[g]   # noqa: E731
            self._rsepoch = torch.zeros(L, dtype=torch.int32, device=self.dev)
            self._sc = []
            for l in range(L):
                st = (ctypes.c_void_p * world)(*[base(g) + self._soff[l] for g in range(world)])
                ar = (ctypes.c_void_p * world)(*[base(g) + self._rcoff + 4 * l for g in range(world)])
                self._sc.append((_lib.Scatter(world, self.rank, ctypes.cast(st, vpp), ctypes.cast(ar, vpp)), st, ar))
        torch.cuda.synchronize()
        dist.barrier()

    def _setup_fused(self):
        L = self.L
        self._epoch = torch.zeros(L, dtype=torch.int32, device=self.dev)
        if self.world == 1:
            self._arrive_local = torch.zeros(L, dtype=torch.int32, device=self.dev)
            own = [self._arrive_local[l:].data_ptr() for l in range(L)]
            peers = [[] for _ in range(L)]
        else:
            own = [self._pbase + self._coff + 4 * l for l in range(L)]
            peers = [[self._peer_base[g] + self._coff + 4 * l for g in self._peers] for l in range(L)]
        n = len(self._peers) if self.world > 1 else 0
        self._ex = []
        for l in range(L):
            pp = (ctypes.c_void_p * max(n, 1))(*([self._peer_base[g] + self._goff[l] for g in self._peers] if n else [0]))
            arr = (ctypes.c_void_p * (n + 1))(*([own[l]] + peers[l]))
            vpp = ctypes.POINTER(ctypes.c_void_p)
            ex = _lib.Exchange(n, ctypes.cast(pp, vpp), ctypes.cast(arr, vpp), own[l], self._epoch[l:].data_ptr(),
                               self.bad.data_ptr())
            self._ex.append((ex, pp, arr))

    def _init_weights(self, seed):
        """Glorot-uniform bounds of the reference init (phantom.py:126-129), drawn on device."""
        s, k, p, off = self.s, self.k, self.p, self.off
        g = torch.Generator(device=self.dev)
        lds, ldk = off["lds"], off["ldk"]
        for jj, j in enumerate(self.local):
            for l in range(self.L):
                g.manual_seed((seed * 1_000_003 + l * 1009 + j) & 0x7FFFFFFF)
                m = self.master[jj, l]
                a = math.sqrt(6.0 / (2 * s))
                m[0:s * lds].view(s, lds)[:, :s].uniform_(-a, a, generator=g)
                a = math.sqrt(6.0 / (s + k))
                m[off["comp"]:off["comp"] + k * lds].view(k, lds)[:, :s].uniform_(-a, a, generator=g)
                if p > 1:
                    m[off["dec"]:off["bias"]].view(p - 1, s, ldk)[:, :, :k].uniform_(-a, a, generator=g)
        self.refresh_compute_copy()

    def refresh_compute_copy(self):
        st = torch.cuda.current_stream().cuda_stream
        for w in self.w:
            self.ctx.call("ppx_cast", _lib.PPX_FP32, self.master.data_ptr(), self.pdt, w.data_ptr(),
                          self.master.numel(), st)

    def load_params(self, rank_layers):
        """Copy reference-format shards (dicts / PhantomLayers, numpy or torch) of this GPU's
        logical ranks into the engine (weights identical to the oracle for parity runs)."""
        s, k, p, off = self.s, self.k, self.p, self.off
        lds, ldk = off["lds"], off["ldk"]
        for jj, j in enumerate(self.local):
            for l in range(self.L):
                lay = rank_layers[j][l]
                get = (lambda nm: lay[nm]) if isinstance(lay, dict) else (lambda nm: getattr(lay, nm))
                m = self.master[jj, l]
                m[0:s * lds].view(s, lds)[:, :s].copy_(torch.as_tensor(get("local"), dtype=torch.float64))
                m[off["comp"]:off["comp"] + k * lds].view(k, lds)[:, :s].copy_(
                    torch.as_tensor(get("compressor"), dtype=torch.float64))
                decs = get("decompressors")
                for q in range(p - 1):
                    i = q + (1 if q >= j else 0)
                    base = off["dec"] + q * s * ldk
                    m[base:base + s * ldk].view(s, ldk)[:, :k].copy_(torch.as_tensor(decs[i], dtype=torch.float64))
                self.bias[jj, l].copy_(torch.as_tensor(get("bias"), dtype=torch.float64))
        self.refresh_compute_copy()

    def layer_views(self, jj, l, master=None, bias=None):
        """Reference-shaped views (local, compressor, {src: decompressor}, bias) of one shard
        (of the fp32 master, or of another flat tensor in the same layout, e.g. Adam moments)."""
        s, k, p, off = self.s, self.k, self.p, self.off
        lds, ldk = off["lds"], off["ldk"]
        m = self.master[jj, l] if master is None else master
        j = self.local[jj]
        decs = {}
        for q in range(p - 1):
            i = q + (1 if q >= j else 0)
            base = off["dec"] + q * s * ldk
            decs[i] = m[base:base + s * ldk].view(s, ldk)[:, :k]
        return {"local": m[0:s * lds].view(s, lds)[:, :s], "compressor": m[off["comp"]:off["comp"] + k * lds]
                .view(k, lds)[:, :s], "decompressors": decs, "bias": self.bias[jj, l] if bias is None else bias}

    def save_checkpoint(self, path, seed: int = 0, *, optimizer_state: bool = False):
        """PSHARD01 checkpoint of the weights (+ optimizer sidecar): every process writes its own
        logical ranks in place (checkpoint.py)."""
        from . import checkpoint
        bar = _dist_barrier if self.world > 1 else None
        fn = checkpoint.save_state if optimizer_state else checkpoint.save_engine
        fn(path, self, seed, create=self.rank == 0, barrier=bar)

    def load_checkpoint(self, path, *, optimizer_state: bool = False) -> int:
        from . import checkpoint
        seed = (checkpoint.load_state if optimizer_state else checkpoint.load_engine)(path, self)
        torch.cuda.synchronize()
        return seed

    # ------------------------------------------------------------------------------------------
    def _layer(self, jj, l, par):
        L = _lib.Layer(self.s, self.k, self.p, self.local[jj], self.w[par][jj, l].data_ptr(),
                       self.master[jj, l].data_ptr(), self.bias[jj, l].data_ptr())
        self._keep.append(L)
        return L

    def _update(self, jj, l, par):
        kind = _lib.PPX_UPDATE_ADAM if self.optimizer == "adam" else _lib.PPX_UPDATE_SGD
        u = _lib.Update(kind, self.hyper.data_ptr(), self.master[jj, l].data_ptr(),
                        self.w[1 - par][jj, l].data_ptr(),
                        self.adam_m[jj, l].data_ptr() if kind == _lib.PPX_UPDATE_ADAM else None,
                        self.adam_v[jj, l].data_ptr() if kind == _lib.PPX_UPDATE_ADAM else None,
                        None, self.bad.data_ptr())
        self._keep.append(u)
        return u

    def _received(self, l, j):
        if self.Hr is not None:
            jj = self.local.index(j)
            return self.Hr[l].data_ptr() + jj * self.B * self.off["ldk"] * self.Hr[l].element_size()
        return self.H[l].data_ptr() + j * self.B * self.off["ldk"] * self.H[l].element_size()

    _KERNEL_CALLS = {"ppx_compress", "ppx_forward_update", "ppx_forward_output", "ppx_error_phantoms", "ppx_wgrad",
                     "ppx_backward_delta", "ppx_optimizer_step", "ppx_compress_n", "ppx_forward_n", "ppx_error_phantoms_n", "ppx_compress_push",
                     "ppx_peer_signal", "ppx_peer_wait", "ppx_peer_push", "ppx_forward_fused",
                     "ppx_error_phantoms_scatter", "ppx_reduce_received", "ppx_backward_fused",
                     "ppx_backward_delta_n"}

    def _call(self, name, *args):
        """ctx.call that counts the launches of our own kernels (NCCL / memsets excluded)."""
        self.ctx.call(name, *args)
        if name in self._KERNEL_CALLS:
            self._launches += 1
            self.trace.append(name)

    @staticmethod
    def _join(src: torch.cuda.Stream, dst: torch.cuda.Stream):
        ev = torch.cuda.Event()
        ev.record(src)
        dst.wait_event(ev)

    def _io(self, jj, l, par, **kw):
        io = _lib.RankIO()
        io.layer = ctypes.pointer(self._layer(jj, l, par))
        for k_, v in kw.items():
            setattr(io, k_, v)
        return io

    def _ios(self, ios):
        arr = (_lib.RankIO * len(ios))(*ios)
        self._keep.append(arr)
        return arr

    def _gh(self, l, h):
        """Phantom buffer of batch half h of layer l ([p, B/H, ldk] at offset h)."""
        Bh = self.B // self.halves
        return self.G[l].data_ptr() + h * self.p * Bh * self.off["ldk"] * self.G[l].element_size()

    def _forward(self, par, S, train=True):
        st, pdt, B, s, R, H = S.cuda_stream, self.pdt, self.B, self.s, self.R, self.halves
        Bh = B // H
        esz = self.Y[par][0][0].element_size()
        rows = lambda t, h: t.data_ptr() + h * Bh * s * esz   # noqa: E731  (row block h of a [B, s] buffer)
        mean = self.reduction == "mean"
        ag_done = {}

        def compress(l, h):
            ios = [self._io(jj, l, par, x=rows(self.Y[par][jj][l], h), ld_x=s) for jj in range(R)]
            if self.p2p == 2:   # compress, then ONE NVLink push kernel (copy to peers + flag)
                n = len(self._peers)
                for c in range(0, R, self.group):
                    self._call("ppx_compress_n", pdt, min(self.group, R - c), self._ios(ios[c:c + self.group]), Bh,
                               self._gh(l, h), st)
                own = self._gh(l, h) + self.rank * R * Bh * self.off["ldk"] * esz
                nbytes = R * Bh * self.off["ldk"] * esz
                off = own - self._pbase
                dst = (ctypes.c_void_p * max(n, 1))(*[self._peer_base[g] + off for g in self._peers])
                self._keep.append(dst)
                self._call("ppx_peer_push", own, nbytes, n, dst, self._sig_dst[l], self._sigcnt[l:].data_ptr(), st)
                return
            if self.p2p:   # fused all-gather: NVLink stores from the epilogue, then the layer flag
                n = len(self._peers)
                for c in range(0, R, self.group):
                    self._call("ppx_compress_push", pdt, min(self.group, R - c), self._ios(ios[c:c + self.group]),
                               Bh, self._gh(l, h), n, self._push_dst[l], st)
                self._call("ppx_peer_signal", n, self._sig_dst[l], self._sigcnt[l:].data_ptr(), st)
                return
            for c in range(0, R, self.group):
                self._call("ppx_compress_n", pdt, min(self.group, R - c), self._ios(ios[c:c + self.group]), Bh,
                           self._gh(l, h), st)
            if self.world > 1 and not self._dbg_skip_ag:
                self._join(S, self.comm_stream)
                self._call("ppx_all_gather", pdt, self._gh(l, h), Bh * self.off["ldk"], R,
                           self.comm_stream.cuda_stream)
                ev = torch.cuda.Event()
                ev.record(self.comm_stream)
                ag_done[(l, h)] = ev

        if self.fused:
            for l in range(self.L):
                last = train and l == self.L - 1
                ios = []
                for jj in range(R):
                    kw = dict(x=self.Y[par][jj][l].data_ptr(), ld_x=s, out=self.Y[par][jj][l + 1].data_ptr(), ld_out=s)
                    if last:
                        kw.update(out=None if self.skip_output else kw["out"], aux=self.D[jj][0].data_ptr(), ld_aux=s,
                                  target=self.Tgt[par][jj].data_ptr(), ld_t=s, colsum=self.gbias[jj, l].data_ptr())
                    ios.append(self._io(jj, l, par, **kw))
                self._call("ppx_forward_fused", pdt, R, self._ios(ios), B, self.act.code, self.G[l].data_ptr(),
                           int(last), 1.0 / B if mean else 1.0, 0.5 / B if mean else 0.5,
                           self.loss.data_ptr() if last else None, ctypes.byref(self._ex[l][0]), st)
            return
        # software pipeline over batch halves: the all-gather of one half overlaps the other
        # half's GEMMs (H = 2 on multi-GPU runs; H = 1 has nothing to hide)
        for h in range(H):
            compress(0, h)
        for l in range(self.L):
            last = train and l == self.L - 1
            for h in range(H):
                if (l, h) in ag_done:
                    S.wait_event(ag_done[(l, h)])
                if self.p2p:
                    self._call("ppx_peer_wait", len(self._peers), self._wait_src[l], self._waitcnt[l:].data_ptr(),
                               self.bad.data_ptr(), st)
                ios = []
                for jj in range(R):
                    kw = dict(x=rows(self.Y[par][jj][l], h), ld_x=s, out=rows(self.Y[par][jj][l + 1], h), ld_out=s)
                    if last:   # the output y itself is never read by the backward pass: not stored
                        kw.update(out=None if self.skip_output else kw["out"], aux=rows(self.D[jj][0], h), ld_aux=s,
                                  target=rows(self.Tgt[par][jj], h), ld_t=s, colsum=self.gbias[jj, l].data_ptr())
                    ios.append(self._io(jj, l, par, **kw))
                for c in range(0, R, self.group):
                    self._call("ppx_forward_n", pdt, min(self.group, R - c), self._ios(ios[c:c + self.group]), Bh,
                               self.act.code, self._gh(l, h), int(last), 1.0 / B if mean else 1.0,
                               0.5 / B if mean else 0.5, self.loss.data_ptr() if last else None, st)
                if l + 1 < self.L:
                    compress(l + 1, h)

    def _launch_wgrad(self, items, st):
        arr = (_lib.WgradItem * len(items))(*items)
        self._keep.append(arr)
        self._call("ppx_wgrad", self.pdt, len(items), arr, st)

    def _backward(self, par, S):
        st, pdt, B, s, R, L = S.cuda_stream, self.pdt, self.B, self.s, self.R, self.L
        slot = B * self.off["ldk"]
        esz = self.H[0].element_size()
        cur = 0
        for l in range(L - 1, -1, -1):
            if getattr(self, "nvrs", False) and self.p2p:
                # NVLink reduce-scatter: the error-compression epilogue copies every peer-owned
                # slot into its owner's staging area; reduced after the weight gradients
                ios = [self._io(jj, l, par, x=self.D[jj][cur].data_ptr(), ld_x=s) for jj in range(R)]
                self._call("ppx_error_phantoms_scatter", pdt, R, self._ios(ios), B, self.H[l].data_ptr(),
                           ctypes.byref(self._sc[l][0]), st)
            elif self.group >= R and not os.environ.get("PPX_K3_PERRANK"):
                # one launch: slot i = sum_{local j != i} delta_j . D_{i->j}, every slot with a
                # contributor overwritten (with R = 1 the own slot has none and stays zero: the
                # reduce-scatter is out of place)
                ios = [self._io(jj, l, par, x=self.D[jj][cur].data_ptr(), ld_x=s) for jj in range(R)]
                self._call("ppx_error_phantoms_n", pdt, R, self._ios(ios), B, self.H[l].data_ptr(), st)
            else:   # PPX_NOGROUP profiling: per-rank launches accumulating into zeroed slots
                self._call("ppx_zero", self.H[l].data_ptr(), self.H[l].numel() * esz, st)
                for jj in range(R):
                    self._call("ppx_error_phantoms", pdt, ctypes.byref(self._layer(jj, l, par)), B,
                               self.D[jj][cur].data_ptr(), s, self.H[l].data_ptr(), 1, st)
            nvrs = getattr(self, "nvrs", False) and self.p2p
            if self.world > 1 and not self._dbg_skip_rs and not nvrs:
                self._join(S, self.comm_stream)
                self._call("ppx_reduce_scatter_to", pdt, self.H[l].data_ptr(), self.Hr[l].data_ptr(), slot, R,
                           self.comm_stream.cuda_stream)
            # weight gradients that do not need r_l, overlapped with the reduce-scatter
            per_rank = []
            for jj in range(R):
                j = self.local[jj]
                items = [_lib.WgradItem(ctypes.pointer(self._layer(jj, l, par)), _lib.GRAD_LOCAL | _lib.GRAD_DEC, B,
                                        self.D[jj][cur].data_ptr(), s, self.Y[par][jj][l].data_ptr(), s,
                                        self.G[l].data_ptr(), None, None, ctypes.pointer(self._update(jj, l, par)),
                                        self.halves)]
                if l < L - 1:   # d compressor of layer l+1 (its r arrived one layer ago)
                    items.append(_lib.WgradItem(ctypes.pointer(self._layer(jj, l + 1, par)), _lib.GRAD_COMP, B,
                                                self.D[jj][cur].data_ptr(), s, self.Y[par][jj][l + 1].data_ptr(), s,
                                                None, self._received(l + 1, j), None,
                                                ctypes.pointer(self._update(jj, l + 1, par))))
                per_rank.append(items)
            if self.bwd_fused and R * (4 if l < L - 1 else 3) <= 15:
                # r_l first (exposed), then weight gradients + recurrence as ONE LPT-scheduled launch
                if self.world > 1 and not nvrs:
                    self._join(self.comm_stream, S)
                if nvrs:
                    own = self.H[l].data_ptr() + self.rank * R * slot * esz
                    self._call("ppx_reduce_received", pdt, R, slot, self.world, self.rank, self._pbase + self._soff[l],
                               own, self.Hr[l].data_ptr(), self._pbase + self._rcoff + 4 * l,
                               self._rsepoch[l:].data_ptr(), self.bad.data_ptr(), st)
                ios = []
                if l > 0:
                    for jj in range(R):
                        j = self.local[jj]
                        ios.append(self._io(jj, l, par, x=self.D[jj][cur].data_ptr(), ld_x=s,
                                            out=self.D[jj][1 - cur].data_ptr(), ld_out=s,
                                            mask=self.Y[par][jj][l].data_ptr() if self.act is Activation.RELU else None,
                                            ld_m=s, received=self._received(l, j),
                                            colsum=self.gbias[jj, l - 1].data_ptr()))
                flat = [it for chunk in per_rank for it in chunk]
                arr = (_lib.WgradItem * len(flat))(*flat)
                self._keep.append(arr)
                self._call("ppx_backward_fused", pdt, len(flat), arr, len(ios), self._ios(ios), B, self.act.code, st)
                if l > 0:
                    cur = 1 - cur
                continue
            nprob = 2 + (1 if l < L - 1 else 0) if self.p > 1 else 1
            per = max(1, min(self.group, 16 // nprob))
            nl = -(-R // per)
            per = -(-R // nl)
            # leave SMs to the reduce-scatter running on the comm stream under these GEMMs
            if self.world > 1 and self.comm_sms:
                self.ctx.call("ppx_set_reserved_sms", self.comm_sms)
            for c in range(0, R, per):
                self._launch_wgrad([it for chunk in per_rank[c:c + per] for it in chunk], st)
            if self.world > 1 and self.comm_sms:
                self.ctx.call("ppx_set_reserved_sms", 0)
            if self.world > 1 and not nvrs:
                self._join(self.comm_stream, S)
            if nvrs:
                own = self.H[l].data_ptr() + self.rank * R * slot * esz
                self._call("ppx_reduce_received", pdt, R, slot, self.world, self.rank, self._pbase + self._soff[l], own,
                           self.Hr[l].data_ptr(), self._pbase + self._rcoff + 4 * l, self._rsepoch[l:].data_ptr(),
                           self.bad.data_ptr(), st)
            if l > 0:
                ios = []
                for jj in range(R):
                    j = self.local[jj]
                    ios.append(self._io(jj, l, par, x=self.D[jj][cur].data_ptr(), ld_x=s,
                                        out=self.D[jj][1 - cur].data_ptr(), ld_out=s,
                                        mask=self.Y[par][jj][l].data_ptr() if self.act is Activation.RELU else None,
                                        ld_m=s, received=self._received(l, j),
                                        colsum=self.gbias[jj, l - 1].data_ptr()))
                for c in range(0, R, self.group):
                    self._call("ppx_backward_delta_n", pdt, min(self.group, R - c), self._ios(ios[c:c + self.group]),
                               B, self.act.code, st)
                cur = 1 - cur
        # d compressor of layer 0, all local ranks in one launch
        items = [_lib.WgradItem(ctypes.pointer(self._layer(jj, 0, par)), _lib.GRAD_COMP, B,
                                self.D[jj][cur].data_ptr(), s, self.Y[par][jj][0].data_ptr(), s, None,
                                self._received(0, self.local[jj]), None, ctypes.pointer(self._update(jj, 0, par)))
                 for jj in range(R)]
        if self.p > 1:
            for c in range(0, R, self.group):
                self._launch_wgrad(items[c:c + self.group], st)
        # biases of all local ranks and layers in one elementwise launch
        kind = _lib.PPX_UPDATE_ADAM if self.optimizer == "adam" else _lib.PPX_UPDATE_SGD
        self._call("ppx_optimizer_step", kind, self.hyper.data_ptr(), self.bias.data_ptr(), self.gbias.data_ptr(),
                   self.adam_bm.data_ptr() if kind == _lib.PPX_UPDATE_ADAM else None,
                   self.adam_bv.data_ptr() if kind == _lib.PPX_UPDATE_ADAM else None,
                   self.bias.numel(), _lib.PPX_FP32, None, self.bad.data_ptr(), st)

    def _step_body(self, par, S):
        self._keep.clear()
        self._launches = 0
        self.trace = []
        c, st = self.ctx, S.cuda_stream
        self._call("ppx_zero", self.gbias.data_ptr(), self.gbias.numel() * 4, st)
        self._call("ppx_zero", self.loss.data_ptr(), 4, st)
        self._forward(par, S)
        self._backward(par, S)
        if self.world > 1:
            self._call("ppx_all_reduce_f32", self.loss.data_ptr(), 1, st)
        self.launch_count = self._launches

    # ------------------------------------------------------------------------------------------
    def _set_hyper(self):
        self.t += 1
        b1, b2 = self.betas
        self.hyper_host.copy_(torch.tensor([self.lr, b1, b2, self.eps, 1 - b1 ** self.t, 1 - b2 ** self.t]))

    def step(self, graph: bool = True):
        """One training iteration on the device-resident batch of the current parity."""
        par = self.parity
        S = torch.cuda.current_stream()
        self._set_hyper()
        self.hyper.copy_(self.hyper_host, non_blocking=True)
        if graph and self.graphs[par] is not None:
            self.graphs[par].replay()
        else:
            self._step_body(par, S)
        self.parity = 1 - par

    def capture(self):
        """Capture one CUDA graph per parity (weights / input double buffers alternate)."""
        torch.cuda.synchronize()
        for par in (0, 1):
            g = torch.cuda.CUDAGraph()
            cs = torch.cuda.Stream(self.dev)
            cs.wait_stream(torch.cuda.current_stream())
            with torch.cuda.graph(g, stream=cs):
                self._step_body(par, torch.cuda.current_stream())
            self.graphs[par] = g
        torch.cuda.synchronize()

    def close(self):
        """Release the CUDA graphs (they hold NCCL work) and then this GPU's communicator.
        Call on every rank at the same point of the program (idempotent)."""
        if self.ctx.handle is None:
            return
        torch.cuda.synchronize()
        for g in self.graphs:
            if g is not None:
                g.reset()
        self.graphs = [None, None]
        torch.cuda.synchronize()
        self.ctx.close()

    def forward_only(self, par=None):
        """Inference (config C5): the forward loop without tape, loss or delta."""
        par = self.parity if par is None else par
        self._forward(par, torch.cuda.current_stream(), train=False)
        return [self.Y[par][jj][self.L] for jj in range(self.R)]

    # ------------------------------------------------------------------------------------------
    def set_batch(self, x_shards, t_shards, par=None):
        """Device tensors (B, s) per local rank -> input/target buffers of a parity."""
        par = self.parity if par is None else par
        for jj in range(self.R):
            self.Y[par][jj][0].copy_(x_shards[jj])
            self.Tgt[par][jj].copy_(t_shards[jj])

    def load_batch_async(self, x_host, t_host, par):
        """H2D of one step's inputs (pinned host [R, B, s] each) on the copy stream; returns the
        event the compute stream must wait on."""
        with torch.cuda.stream(self.copy_stream):
            for jj in range(self.R):
                self.Y[par][jj][0].copy_(x_host[jj], non_blocking=True)
                self.Tgt[par][jj].copy_(t_host[jj], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.copy_stream)
        return ev

    def read_loss(self) -> float:
        self.out_host.copy_(self.loss, non_blocking=True)
        self.bad_host.copy_(self.bad, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        if int(self.bad_host[0]) & 2:
            raise TrainingError("a peer GPU never published its phantoms (NVLink exchange / fused wait timed out)")
        if int(self.bad_host[0]) != 0:
            raise TrainingError("non-finite gradient detected on the device")
        return float(self.out_host[0].item())

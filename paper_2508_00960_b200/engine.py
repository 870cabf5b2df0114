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

from . import _lib, kernels, schedule
from .core import Activation, as_activation, flat_offsets
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
                 dtype: torch.dtype = torch.bfloat16, seed: int = 0, ctx: _lib.Context | None = None,
                 fused: bool | None = None, nvrs: bool | None = None, group: int | None = None,
                 bwd_fused: bool | None = None, k3_fused: bool | None = None, store_output: bool = False,
                 capture: bool = False, mask_bits: bool | None = None):
        """Launch-plan switches (None = the default plan; every plan computes the same step):

        fused      compression + phantom all-gather + forward of a layer as ONE launch (bf16, s and k
                   multiples of 64, <= 8 logical ranks per GPU); otherwise compression, NCCL
                   all-gather on the comm stream, then the K-concatenated forward GEMM.
        nvrs       (world > 1, bf16, k % 8 == 0) reduce-scatter through NVLink peer memory from the
                   error-compression epilogue instead of NCCL; default when a GPU owns >= 2 ranks.
        group      logical ranks per grouped launch (default all R; 1 = the per-GPU launch shapes of
                   a run with one logical rank per GPU, on one GPU).
        k3_fused   error compression + weight gradients of a layer as one LPT-scheduled launch
                   (error tiles first), then the recurrence once r_l is in: the NVLink
                   reduce-scatter runs under the weight gradients.  Default when a launch holds
                   one logical rank (world > 1 with nvrs and <= 2 ranks per GPU, or group=1).
        bwd_fused  weight gradients + error recurrence of a layer as one LPT-scheduled launch per
                   group (the plan before k3_fused; used when k3_fused is off).
        store_output  keep the output layer's y (training steps never read it back).
        mask_bits  the forward epilogue also stores ReLU'(pre) of every inner layer as a bit mask
                   and the recurrence reads it instead of the bf16 activations (1/16 of the mask
                   bytes); default for bf16 ReLU with s % 64 == 0.
        capture    keep the raw weight gradients (fp32, flat layout) and every layer's delta of the
                   last eager step (parity tests; CUDA-graph replays do not refresh the deltas).
        """
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
        if world > 1 and not self._dist_ready():
            raise ConfigurationError("world > 1 needs torch.distributed initialised (IPC handles and barriers)")
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
        self.capture_grads = capture
        self.grad = torch.zeros_like(self.master) if capture else None
        self.deltas = [None] * L            # capture: deltas[l][jj] = delta_l of the last eager step
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
        bits_ok = dtype == torch.bfloat16 and self.act is Activation.RELU and s % 64 == 0 and layers > 1
        if mask_bits and not bits_ok:
            raise ConfigurationError("bit masks need bf16, ReLU and s % 64 == 0")
        self.mask_bits = bits_ok if mask_bits is None else bool(mask_bits)
        # bits[jj][l] = ReLU'(pre_{l-1}) = (Y[l] > 0) packed 32 per int32 word, l = 1 .. L-1
        self.bits = ([[None] + [torch.zeros((B, s // 32), dtype=torch.int32, device=self.dev) for _ in range(1, layers)]
                      for _ in range(R)] if self.mask_bits else None)
        self.bad = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.group = R if group is None else max(1, min(int(group), R))
        auto_fused = (dtype == torch.bfloat16 and s % 64 == 0 and k % 64 == 0 and R <= 8 and self.group == R)
        if fused and not auto_fused:
            raise ConfigurationError("fused forward needs bf16, s and k multiples of 64, <= 8 ranks per GPU and "
                                     "one group per layer")
        self.fused = auto_fused if fused is None else bool(fused)
        # NVLink reduce-scatter (world > 1, bf16): default when a GPU owns >= 2 logical ranks (C3 on
        # 4 GPUs: 5.41 -> 5.31 ms); with one rank per GPU the NCCL reduce-scatter on the comm stream
        # under the weight gradients is faster (C2 on 4 GPUs: 2.53 -> 2.70 ms)
        nvrs_ok = world > 1 and dtype == torch.bfloat16 and R <= 8 and k % 8 == 0
        if nvrs and not nvrs_ok:
            raise ConfigurationError("NVLink reduce-scatter needs world > 1, bf16, <= 8 ranks per GPU and k % 8 == 0")
        self.nvrs = nvrs_ok if nvrs is None else bool(nvrs)
        # IPC-shared phantom / staging region (world > 1): needed by the fused forward's in-kernel
        # all-gather and by the NVLink reduce-scatter
        self.p2p = world > 1 and (self.fused or self.nvrs)
        if self.p2p:
            self._setup_p2p(dtype)
        else:
            self.G = [torch.zeros((p, B, ldk), dtype=dtype, device=self.dev) for _ in range(L)]
        if self.fused:
            self._setup_fused()
        self.H = [torch.zeros((p, B, ldk), dtype=dtype, device=self.dev) for _ in range(L)]
        # out-of-place reduce-scatter target (world > 1): this GPU's R received slots
        self.Hr = [torch.zeros((R, B, ldk), dtype=dtype, device=self.dev) for _ in range(L)] if world > 1 else None
        self.loss = torch.zeros(1, dtype=f32, device=self.dev)
        self.fence = torch.zeros(1, dtype=f32, device=self.dev)
        # optimizer scalars [lr, beta1, beta2, eps, 1 - beta1^t, 1 - beta2^t]: the bias corrections
        # are advanced on the device by the first launch of every step (graph replays need no host
        # write, and no pinned buffer is rewritten while an earlier copy of it may be in flight)
        b1, b2 = betas
        self.hyper = torch.tensor([lr, b1, b2, eps, 0.0, 0.0], dtype=f32, device=self.dev)
        self.tdev = torch.zeros(1, dtype=torch.int32, device=self.dev)
        self.out_host = torch.zeros(1, dtype=f32).pin_memory()
        self.bad_host = torch.zeros(1, dtype=torch.int32).pin_memory()
        # loss_async(): ring of pinned (loss, flag) slots for reads that lag the steps
        self._loss_ring = [(torch.zeros(1, dtype=f32).pin_memory(), torch.zeros(1, dtype=torch.int32).pin_memory())
                           for _ in range(4)]
        self._loss_i = 0
        if dtype == torch.float32:   # 3xTF32 hi/lo splits: reserve so graph capture never allocates
            per_call = 4 * B * s + 2 * p * B * ldk + 2 * T + 4 * s * ldk
            self.ctx.call("ppx_reserve_workspace", int(2 * 4 * per_call * 1.25) + (1 << 20))
        self.graphs = [None, None]
        self.infer_graphs = [None, None]
        self.infer_launch_count = 0
        self.parity = 0
        self.skip_output = not store_output
        # weight gradients + error recurrence of a layer as one LPT-scheduled launch (after the
        # reduce-scatter): default when a launch holds one logical rank, where either launch alone
        # leaves ~1.4 rounds of tiles
        # (<= 16 problems per launch: 4 per logical rank)
        auto_bf = dtype == torch.bfloat16 and self.group == 1 and (world > 1 or R > 1)
        if bwd_fused and (dtype != torch.bfloat16 or self.group > 3):
            raise ConfigurationError("fused backward needs bf16 and <= 3 logical ranks per launch group")
        self.bwd_fused = auto_bf if bwd_fused is None else bool(bwd_fused)
        # error compression + weight gradients in one launch (<= 16 problems: p slots, or p/2 slot
        # pairs, + 3 per rank)
        pairs = p % 2 == 0 and k % 64 == 0 and (self.group % 2 == 0 or self.group == 1)
        n_err = p // 2 if pairs else p
        k3_ok = (dtype == torch.bfloat16 and p > 1 and n_err + 3 * self.group <= 16 and
                 ((world > 1 and self.nvrs and self.group == R) or (world == 1 and self.group < R)))
        if k3_fused and not k3_ok:
            raise ConfigurationError("fused error compression + weight gradients needs bf16, p + 3 ranks per launch "
                                     "<= 16 and either the NVLink reduce-scatter or one GPU with per-group launches")
        # default with <= 2 ranks per launch, and on every multi-GPU run the limit admits (C3 at
        # N = 2: 4 slot pairs + 4 ranks x 3 = 16 problems)
        self.k3_fused = (k3_ok and (self.group <= 2 or world > 1)) if k3_fused is None else bool(k3_fused)
        if self.k3_fused:
            self.bwd_fused = False
        # one GPU with every logical rank in one launch group: the error compression (p/2 slot-pair
        # problems) rides in the first weight-gradient launch of the layer, error tiles first
        # (<= 16 problems per launch; PPX_NO_K3G=1 keeps its own launch, A/B only)
        self.k3_grouped = (not self.k3_fused and not self.bwd_fused and world == 1 and R > 1 and R % 2 == 0
                           and self.group >= R and dtype == torch.bfloat16 and p % 2 == 0 and k % 64 == 0
                           and not os.environ.get("PPX_NO_K3G"))
        # layer-0 compressor gradient with the batch split (ppx_wgrad_splitk): fp32 partial sums
        # (PPX_NO_SPLITK=1 keeps the one-launch form, A/B only)
        self.splitk_off = bool(os.environ.get("PPX_NO_SPLITK"))
        nparts = max((c1 - c0) * self._layer0_split(c1 - c0) for c0, c1 in self._chunks()) if p > 1 else 0
        self.splitk_parts = torch.zeros(max(1, nparts * k * self.off["lds"]), dtype=f32, device=self.dev)
        self._keep = []   # ctypes structs of the launch being built
        self.launch_count = 0
        self.trace = []   # kernel-launching ABI calls of the last step body (profiling labels)
        self._timing = None   # per-launch CUDA events (profile_step)
        # algorithmic GEMM FLOPs per logical rank of each contraction
        self._f_compress = 2 * B * s * k
        self._f_forward = 2 * B * s * (s + (p - 1) * k)
        self._f_error = 2 * B * s * (p - 1) * k
        self._f_recurrence = 2 * B * s * (s + k)

    # ------------------------------------------------------------------------------------------
    @staticmethod
    def _dist_ready():
        import torch.distributed as dist
        return dist.is_available() and dist.is_initialized()

    def _setup_p2p(self, dtype):
        """IPC region on every GPU, mapped by all peers (handles exchanged over torch.distributed):
        [L][p, B, ldk] phantoms | [L] fused-forward arrival counters | [L] reduce-scatter arrival
        counters | [L][world, R, B, ldk] reduce-scatter staging.  Identical layouts, so a peer
        address is peer_base + (local address - local base)."""
        import torch.distributed as dist
        p, B, L, ldk, world = self.p, self.B, self.L, self.off["ldk"], self.world
        esz = torch.tensor([], dtype=dtype).element_size()
        gbytes = p * B * ldk * esz
        self._goff = [l * gbytes for l in range(L)]
        self._coff = L * gbytes                                           # per-layer arrival counters
        self._rcoff = self._coff + ((L * 4 + 255) // 256) * 256           # reduce-scatter arrival counters
        sbytes = world * self.R * B * ldk * esz if self.nvrs else 0       # reduce-scatter staging per layer
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

    def phantoms_view(self, l):
        """[p, B, k] view of layer l's gathered phantoms (slot i = logical rank i's g_i)."""
        return self.G[l][:, :, :self.k]

    def received_view(self, l, jj):
        """[B, k] view of the error phantoms r_j local rank jj received for layer l."""
        if self.Hr is not None:
            return self.Hr[l][jj, :, :self.k]
        return self.H[l][self.local[jj], :, :self.k]

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
                        self.grad[jj, l].data_ptr() if self.capture_grads else None, self.bad.data_ptr())
        self._keep.append(u)
        return u

    def _received(self, l, j):
        if self.Hr is not None:
            jj = self.local.index(j)
            return self.Hr[l].data_ptr() + jj * self.B * self.off["ldk"] * self.Hr[l].element_size()
        return self.H[l].data_ptr() + j * self.B * self.off["ldk"] * self.H[l].element_size()

    _KERNEL_CALLS = {"ppx_compress", "ppx_forward_update", "ppx_forward_output", "ppx_error_phantoms", "ppx_wgrad",
                     "ppx_backward_delta", "ppx_optimizer_step", "ppx_compress_n", "ppx_forward_n",
                     "ppx_error_phantoms_n", "ppx_forward_fused", "ppx_error_phantoms_scatter", "ppx_reduce_received",
                     "ppx_backward_fused", "ppx_backward_delta_n", "ppx_hyper_advance",
                     "ppx_backward_wgrad_errors", "ppx_wgrad_splitk"}

    def _call(self, name, *args, flops=0):
        """ctx.call that records the kernel-launching ABI calls of the step (`trace`, the labels
        of ncu launch lists); under profile_step() every such call is bracketed by CUDA events on
        its stream and tagged with its algorithmic GEMM FLOPs.  Kernel counts come from the
        library itself (ppx_kernel_launches)."""
        timed = self._timing is not None and name in self._KERNEL_CALLS
        if timed:
            e0 = torch.cuda.Event(enable_timing=True)
            e0.record()
        self.ctx.call(name, *args)
        if timed:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record()
            self._timing.append((name, e0, e1, flops))
        if name in self._KERNEL_CALLS:
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

    def _chunks(self):
        """Local-rank index ranges of the grouped launches."""
        return [(c, min(c + self.group, self.R)) for c in range(0, self.R, self.group)]

    def _forward(self, par, S, train=True):
        st, pdt, B, s, R = S.cuda_stream, self.pdt, self.B, self.s, self.R
        mean = self.reduction == "mean"

        def ios_for(l, last):
            ios = []
            for jj in range(R):
                kw = dict(x=self.Y[par][jj][l].data_ptr(), ld_x=s, out=self.Y[par][jj][l + 1].data_ptr(), ld_out=s)
                if last:   # the output y itself is never read by the backward pass: not stored
                    kw.update(out=None if self.skip_output else kw["out"], aux=self.D[jj][0].data_ptr(), ld_aux=s,
                              target=self.Tgt[par][jj].data_ptr(), ld_t=s, colsum=self.gbias[jj, l].data_ptr())
                elif train and self.mask_bits:   # the recurrence of layer l+1 masks with these bits
                    kw.update(bits=self.bits[jj][l + 1].data_ptr(), ld_bits=s // 32)
                ios.append(self._io(jj, l, par, **kw))
            return ios

        scales = lambda last: (1.0 / B if mean else 1.0, 0.5 / B if mean else 0.5,   # noqa: E731
                               self.loss.data_ptr() if last else None)
        if self.fused:
            for l in range(self.L):
                last = train and l == self.L - 1
                self._call("ppx_forward_fused", pdt, R, self._ios(ios_for(l, last)), B, self.act.code,
                           self.G[l].data_ptr(), int(last), *scales(last), ctypes.byref(self._ex[l][0]), st,
                           flops=R * (self._f_compress + self._f_forward))
            if not train and self.world > 1:
                # inference ends without the loss all-reduce that orders training steps across
                # GPUs: fence here so the next call's phantom stores never reach a peer that is
                # still reading this call's phantoms
                self._call("ppx_all_reduce_f32", self.fence.data_ptr(), 1, st)
            return
        for l in range(self.L):
            last = train and l == self.L - 1
            ios = [self._io(jj, l, par, x=self.Y[par][jj][l].data_ptr(), ld_x=s) for jj in range(R)]
            for c0, c1 in self._chunks():
                self._call("ppx_compress_n", pdt, c1 - c0, self._ios(ios[c0:c1]), B, self.G[l].data_ptr(), st,
                           flops=(c1 - c0) * self._f_compress)
            if self.world > 1:   # NCCL in-place all-gather of the contiguous phantom slots
                self._join(S, self.comm_stream)
                self._call("ppx_all_gather", pdt, self.G[l].data_ptr(), B * self.off["ldk"], R,
                           self.comm_stream.cuda_stream)
                self._join(self.comm_stream, S)
            ios = ios_for(l, last)
            for c0, c1 in self._chunks():
                self._call("ppx_forward_n", pdt, c1 - c0, self._ios(ios[c0:c1]), B, self.act.code,
                           self.G[l].data_ptr(), int(last), *scales(last), st, flops=(c1 - c0) * self._f_forward)

    def _f_item(self, it):
        """FLOPs of one weight-gradient request (d local 2Bs^2, d decompressors 2Bs(p-1)k,
        d compressor 2Bsk)."""
        B, s, k, p = self.B, self.s, self.k, self.p
        f = 2 * B * s * s if it.parts & _lib.GRAD_LOCAL else 0
        if p > 1:
            f += 2 * B * s * (p - 1) * k if it.parts & _lib.GRAD_DEC else 0
            f += 2 * B * s * k if it.parts & _lib.GRAD_COMP else 0
        return f

    def _layer0_split(self, n_items):
        """Batch chunks of the layer-0 compressor gradient (schedule.layer0_split); 1 = unsplit."""
        return 1 if self.splitk_off else schedule.layer0_split(n_items, self.k, self.s, self.B)

    def _launch_wgrad(self, items, st):
        arr = (_lib.WgradItem * len(items))(*items)
        self._keep.append(arr)
        self._call("ppx_wgrad", self.pdt, len(items), arr, st, flops=sum(self._f_item(it) for it in items))

    def _recurrence_io(self, jj, l, par, cur):
        """[delta | r].[L ; C] -> delta_{l-1} with the ReLU'-mask and d-bias epilogue."""
        kw = dict(bits=self.bits[jj][l].data_ptr(), ld_bits=self.s // 32) if self.mask_bits else {}
        return self._io(jj, l, par, x=self.D[jj][cur].data_ptr(), ld_x=self.s, out=self.D[jj][1 - cur].data_ptr(),
                        ld_out=self.s, mask=self.Y[par][jj][l].data_ptr() if self.act is Activation.RELU else None,
                        ld_m=self.s, received=self._received(l, self.local[jj]),
                        colsum=self.gbias[jj, l - 1].data_ptr(), **kw)

    def _backward(self, par, S):
        st, pdt, B, s, R, L = S.cuda_stream, self.pdt, self.B, self.s, self.R, self.L
        slot = B * self.off["ldk"]
        esz = self.H[0].element_size()
        nvrs = self.nvrs
        cur = 0
        for l in range(L - 1, -1, -1):
            if self.capture_grads:
                self.deltas[l] = [self.D[jj][cur].clone() for jj in range(R)]
            ios = [self._io(jj, l, par, x=self.D[jj][cur].data_ptr(), ld_x=s) for jj in range(R)]
            if self.k3_fused or self.k3_grouped:
                pass                      # error compression runs inside the weight-gradient launch
            elif nvrs:
                # NVLink reduce-scatter: the error-compression epilogue copies every peer-owned
                # slot into its owner's staging area; reduced after the weight gradients
                self._call("ppx_error_phantoms_scatter", pdt, R, self._ios(ios), B, self.H[l].data_ptr(),
                           ctypes.byref(self._sc[l][0]), st, flops=R * self._f_error)
            elif self.group >= R:
                # one launch: slot i = sum_{local j != i} delta_j . D_{i->j}, every slot with a
                # contributor overwritten (with R = 1 the own slot has none and stays zero: the
                # reduce-scatter is out of place)
                self._call("ppx_error_phantoms_n", pdt, R, self._ios(ios), B, self.H[l].data_ptr(), st,
                           flops=R * self._f_error)
            else:   # per-group launches accumulate into zeroed slots
                self._call("ppx_zero", self.H[l].data_ptr(), self.H[l].numel() * esz, st)
                for jj in range(R):
                    self._call("ppx_error_phantoms", pdt, ctypes.byref(self._layer(jj, l, par)), B,
                               self.D[jj][cur].data_ptr(), s, self.H[l].data_ptr(), 1, st, flops=self._f_error)
            if self.world > 1 and not nvrs and not self.k3_fused:
                self._join(S, self.comm_stream)
                self._call("ppx_reduce_scatter_to", pdt, self.H[l].data_ptr(), self.Hr[l].data_ptr(), slot, R,
                           self.comm_stream.cuda_stream)
            # weight gradients that do not need r_l, overlapped with the reduce-scatter
            per_rank = []
            for jj in range(R):
                j = self.local[jj]
                items = [_lib.WgradItem(ctypes.pointer(self._layer(jj, l, par)), _lib.GRAD_LOCAL | _lib.GRAD_DEC, B,
                                        self.D[jj][cur].data_ptr(), s, self.Y[par][jj][l].data_ptr(), s,
                                        self.G[l].data_ptr(), None, None, ctypes.pointer(self._update(jj, l, par)), 1)]
                if l < L - 1:   # d compressor of layer l+1 (its r arrived one layer ago)
                    items.append(_lib.WgradItem(ctypes.pointer(self._layer(jj, l + 1, par)), _lib.GRAD_COMP, B,
                                                self.D[jj][cur].data_ptr(), s, self.Y[par][jj][l + 1].data_ptr(), s,
                                                None, self._received(l + 1, j), None,
                                                ctypes.pointer(self._update(jj, l + 1, par)), 1))
                per_rank.append(items)

            def reduce_received():
                if self.world > 1 and not nvrs:
                    self._join(self.comm_stream, S)
                if nvrs:
                    own = self.H[l].data_ptr() + self.rank * R * slot * esz
                    self._call("ppx_reduce_received", pdt, R, slot, self.world, self.rank, self._pbase + self._soff[l],
                               own, self.Hr[l].data_ptr(), self._pbase + self._rcoff + 4 * l,
                               self._rsepoch[l:].data_ptr(), self.bad.data_ptr(), st)

            if self.k3_fused:
                # error compression + weight gradients as ONE launch per group (error tiles first;
                # with nvrs their epilogue stores peer-owned slots into the owners' staging areas,
                # so the exchange runs under the weight gradients), then r_l, then the recurrence
                if self.world == 1:
                    self._call("ppx_zero", self.H[l].data_ptr(), self.H[l].numel() * esz, st)
                for c0, c1 in self._chunks():
                    flat = [it for chunk in per_rank[c0:c1] for it in chunk]
                    arr = (_lib.WgradItem * len(flat))(*flat)
                    self._keep.append(arr)
                    sc = ctypes.byref(self._sc[l][0]) if self.world > 1 else None
                    self._call("ppx_backward_wgrad_errors", pdt, len(flat), arr, c1 - c0, self._ios(ios[c0:c1]), B,
                               self.H[l].data_ptr(), sc, int(self.world == 1), st,
                               flops=sum(self._f_item(it) for it in flat) + (c1 - c0) * self._f_error)
                reduce_received()
                if l > 0:
                    rios = [self._recurrence_io(jj, l, par, cur) for jj in range(R)]
                    for c0, c1 in self._chunks():
                        self._call("ppx_backward_delta_n", pdt, c1 - c0, self._ios(rios[c0:c1]), B, self.act.code, st,
                                   flops=(c1 - c0) * self._f_recurrence)
                    cur = 1 - cur
                continue
            if self.bwd_fused:
                # r_l first (exposed), then weight gradients + recurrence of each group as ONE
                # LPT-scheduled launch
                reduce_received()
                for c0, c1 in self._chunks():
                    flat = [it for chunk in per_rank[c0:c1] for it in chunk]
                    ios = [self._recurrence_io(jj, l, par, cur) for jj in range(c0, c1)] if l > 0 else []
                    arr = (_lib.WgradItem * len(flat))(*flat)
                    self._keep.append(arr)
                    self._call("ppx_backward_fused", pdt, len(flat), arr, len(ios), self._ios(ios) if ios else None,
                               B, self.act.code, st,
                               flops=sum(self._f_item(it) for it in flat) + len(ios) * self._f_recurrence)
                if l > 0:
                    cur = 1 - cur
                continue
            nprob = 2 + (1 if l < L - 1 else 0) if self.p > 1 else 1
            for i, (c0, c1) in enumerate(schedule.wgrad_launch_chunks(R, self.p, nprob, self.group,
                                                                       self.k3_grouped)):
                flat = [it for chunk in per_rank[c0:c1] for it in chunk]
                if i == 0 and self.k3_grouped:
                    # error compression of all R ranks + the weight gradients of the first ranks
                    arr = (_lib.WgradItem * len(flat))(*flat)
                    self._keep.append(arr)
                    self._call("ppx_backward_wgrad_errors", pdt, len(flat), arr, R, self._ios(ios), B,
                               self.H[l].data_ptr(), None, 0, st,
                               flops=sum(self._f_item(it) for it in flat) + R * self._f_error)
                else:
                    self._launch_wgrad(flat, st)
            reduce_received()
            if l > 0:
                ios = [self._recurrence_io(jj, l, par, cur) for jj in range(R)]
                for c0, c1 in self._chunks():
                    self._call("ppx_backward_delta_n", pdt, c1 - c0, self._ios(ios[c0:c1]), B, self.act.code, st,
                               flops=(c1 - c0) * self._f_recurrence)
                cur = 1 - cur
        # d compressor of layer 0, all local ranks in one launch
        items = [_lib.WgradItem(ctypes.pointer(self._layer(jj, 0, par)), _lib.GRAD_COMP, B,
                                self.D[jj][cur].data_ptr(), s, self.Y[par][jj][0].data_ptr(), s, None,
                                self._received(0, self.local[jj]), None, ctypes.pointer(self._update(jj, 0, par)), 1)
                 for jj in range(R)]
        if self.p > 1:
            for c0, c1 in self._chunks():
                nsplit = self._layer0_split(c1 - c0)
                if nsplit > 1:   # a few long k x s tiles over K = B: split the batch, sum + update after
                    arr = (_lib.WgradItem * (c1 - c0))(*items[c0:c1])
                    self._keep.append(arr)
                    self._call("ppx_wgrad_splitk", pdt, c1 - c0, arr, nsplit, self.splitk_parts.data_ptr(), st,
                               flops=sum(self._f_item(it) for it in items[c0:c1]))
                else:
                    self._launch_wgrad(items[c0:c1], st)
        # biases of all local ranks and layers in one elementwise launch
        kind = _lib.PPX_UPDATE_ADAM if self.optimizer == "adam" else _lib.PPX_UPDATE_SGD
        self._call("ppx_optimizer_step", kind, self.hyper.data_ptr(), self.bias.data_ptr(), self.gbias.data_ptr(),
                   self.adam_bm.data_ptr() if kind == _lib.PPX_UPDATE_ADAM else None,
                   self.adam_bv.data_ptr() if kind == _lib.PPX_UPDATE_ADAM else None,
                   self.bias.numel(), _lib.PPX_FP32, None, self.bad.data_ptr(), st)

    def _step_body(self, par, S):
        self._keep.clear()
        self.trace = []
        k0 = self.ctx.kernel_launches
        st = S.cuda_stream
        nvtx = torch.cuda.nvtx
        nvtx.range_push(f"ppx.step[par={par}]")   # host-side NVTX ranges (ncu --nvtx / nsys filters)
        self._tf32_scope(1, st)
        self._call("ppx_hyper_advance", self.hyper.data_ptr(), self.tdev.data_ptr(), float(self.betas[0]),
                   float(self.betas[1]), st)
        self._call("ppx_zero", self.gbias.data_ptr(), self.gbias.numel() * 4, st)
        self._call("ppx_zero", self.loss.data_ptr(), 4, st)
        nvtx.range_push("ppx.forward")
        self._forward(par, S)
        nvtx.range_pop()
        nvtx.range_push("ppx.backward")
        self._backward(par, S)
        nvtx.range_pop()
        if self.world > 1:
            self._call("ppx_all_reduce_f32", self.loss.data_ptr(), 1, st)
        self._tf32_scope(0, st)
        self.launch_count = self.ctx.kernel_launches - k0   # every kernel the step enqueued
        nvtx.range_pop()

    def _tf32_scope(self, on, st):
        """FP32 tier: inside one step every GEMM operand's 3xTF32 low part is split once and reused
        across calls (ppx_tf32_scope); nothing but ppx calls writes engine buffers in a step."""
        if self.dtype == torch.float32:
            self.ctx.call("ppx_tf32_scope", int(on), st)

    # ------------------------------------------------------------------------------------------
    def set_step_count(self, t: int):
        """Set the optimizer step counter (Adam's t; the next step uses t + 1), e.g. on resume."""
        torch.cuda.synchronize()
        self.t = int(t)
        self.tdev.fill_(int(t))
        torch.cuda.synchronize()

    def set_lr(self, lr: float):
        """Change the learning rate between steps (synchronous: graph replays read it from HBM)."""
        torch.cuda.synchronize()
        self.lr = lr
        self.hyper[0] = lr
        torch.cuda.synchronize()

    def step(self, graph: bool = True):
        """One training iteration on the device-resident batch of the current parity.  Fully
        asynchronous: nothing on the host is rewritten per step (the Adam step counter lives on
        the device), so steps may be issued back to back without reading the loss."""
        par = self.parity
        S = torch.cuda.current_stream()
        self.t += 1
        if graph and self.graphs[par] is not None:
            self.graphs[par].replay()
        else:
            self._step_body(par, S)
        self.parity = 1 - par

    def profile_step(self):
        """One eager step with CUDA events around every kernel launch: returns
        [(abi_call, milliseconds, algorithmic GEMM FLOPs)] in launch order (bench.py's per-kernel
        roofline)."""
        self._timing = []
        try:
            # hold the stream for ~0.1 s so the host enqueues the whole step before the GPU starts
            # it: the event pairs then bracket kernels running back to back, never host gaps
            torch.cuda._sleep(200_000_000)
            self.step(graph=False)
            torch.cuda.synchronize()
            return [(nm, a.elapsed_time(b), f) for nm, a, b, f in self._timing]
        finally:
            self._timing = None

    def capture(self):
        """Capture one CUDA graph per parity (weights / input double buffers alternate)."""
        if self.capture_grads:
            raise ConfigurationError("deltas are recorded by eager steps only: set capture_grads = False first")
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
        for g in self.graphs + self.infer_graphs:
            if g is not None:
                g.reset()
        self.graphs = [None, None]
        self.infer_graphs = [None, None]
        torch.cuda.synchronize()
        self.ctx.close()

    def forward_only(self, par=None, graph=False):
        """Inference (config C5; the reference's loop of pp_forward_layer, test_phantom.py:66-71):
        the forward pass without tape, loss or delta on the input buffers of parity `par`.
        Returns the [B, s] outputs of this GPU's logical ranks (views, overwritten by the next
        call).  graph=True replays the inference graph of capture_inference()."""
        par = self.parity if par is None else par
        if graph and self.infer_graphs[par] is not None:
            self.infer_graphs[par].replay()
        else:
            self._keep.clear()
            st = torch.cuda.current_stream()
            k0 = self.ctx.kernel_launches
            self._tf32_scope(1, st.cuda_stream)
            self._forward(par, st, train=False)
            self._tf32_scope(0, st.cuda_stream)
            self.infer_launch_count = self.ctx.kernel_launches - k0
        return [self.Y[par][jj][self.L] for jj in range(self.R)]

    def capture_inference(self):
        """Capture the forward-only pass of each parity in a CUDA graph."""
        torch.cuda.synchronize()
        for par in (0, 1):
            g = torch.cuda.CUDAGraph()
            cs = torch.cuda.Stream(self.dev)
            cs.wait_stream(torch.cuda.current_stream())
            with torch.cuda.graph(g, stream=cs):
                self._keep.clear()
                st = torch.cuda.current_stream()
                k0 = self.ctx.kernel_launches
                self._tf32_scope(1, st.cuda_stream)
                self._forward(par, st, train=False)
                self._tf32_scope(0, st.cuda_stream)
                self.infer_launch_count = self.ctx.kernel_launches - k0
            self.infer_graphs[par] = g
        torch.cuda.synchronize()

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

    @staticmethod
    def _check_flag(flag: int):
        if flag & 2:
            raise TrainingError("a peer GPU never published its phantoms (NVLink exchange / fused wait timed out)")
        if flag != 0:
            raise TrainingError("non-finite gradient detected on the device")

    def read_loss(self) -> float:
        self.out_host.copy_(self.loss, non_blocking=True)
        self.bad_host.copy_(self.bad, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        self._check_flag(int(self.bad_host[0]))
        return float(self.out_host[0].item())

    def loss_async(self):
        """Enqueue the D2H read of the last step's loss (and non-finite flag) on the current
        stream without waiting; returns a function that waits for that copy only and returns the
        loss (raising TrainingError like read_loss).  A training loop that calls it after step i
        and resolves it after enqueuing step i + 1 keeps the GPU fed while still reading every
        step's loss.  At most 4 reads may be pending at once."""
        self._loss_i = (self._loss_i + 1) % len(self._loss_ring)
        lh, bh = self._loss_ring[self._loss_i]
        lh.copy_(self.loss, non_blocking=True)
        bh.copy_(self.bad, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()

        def result() -> float:
            ev.synchronize()
            self._check_flag(int(bh[0]))
            return float(lh[0].item())
        return result

"""torch.autograd bindings of the phantom layer.

* AllGatherFunction — Algorithm 1 of arXiv 2508.00960 (reference
  collectives.py:115-127): forward all-gathers the k x B phantom shards in ascending rank order,
  backward reduce-scatters the incoming gradient (its adjoint).  `comm` is the in-process
  Communicator of collectives.py (one rank per thread); DistAllGatherFunction is the same pair
  over a torch.distributed process group (NCCL, one process per GPU).

* PhantomLinearFunction — one fused phantom layer: forward is pp_forward_layer (a3: local +
  compress + all-gather + decompress, bias and activation in the GEMM epilogue), backward is
  a7 + a8 + a9 (error phantoms + reduce-scatter, the grouped parameter-gradient launch, and the
  input gradient L^T delta + C^T r).  The layer's parameters are ONE leaf tensor, its flat fp32
  master in PSHARD01 order; its .grad is the flat gradient block (phantom.grads_from_flat views).

  Autograd's incoming gradient is dL/dy; the activation derivative of THIS layer is applied in
  this backward (delta = dL/dy * act'(preact)), so the input gradient is returned without any
  mask, exactly the composition the reference's pp_iteration performs (training.py:195-212).
"""

from __future__ import annotations


import torch

from . import kernels
from .collectives import Direction
from .core import Activation, as_activation
from .errors import ConfigurationError
from .phantom import (PhantomLayer, _native, pp_backward_layer, pp_exchange_error_phantoms, pp_forward_layer,
                      pp_param_grads)


class AllGatherFunction(torch.autograd.Function):
    """y = all_gather(x) over ranks (concatenated along dim 0); dx = reduce_scatter(dy)."""

    @staticmethod
    def forward(ctx, local, comm, rank, layer_index=None):
        ctx.comm, ctx.rank, ctx.layer_index = comm, rank, layer_index
        return comm.all_gather(rank, local, direction=Direction.FORWARD, layer=layer_index)

    @staticmethod
    def backward(ctx, grad):
        g = ctx.comm.reduce_scatter(ctx.rank, grad.contiguous(), direction=Direction.BACKWARD, layer=ctx.layer_index)
        return g, None, None, None


def all_gather(local: torch.Tensor, comm, rank: int, layer_index=None) -> torch.Tensor:
    return AllGatherFunction.apply(local, comm, rank, layer_index)


class DistAllGatherFunction(torch.autograd.Function):
    """The same adjoint pair over torch.distributed (all_gather_into_tensor / reduce_scatter_tensor)."""

    @staticmethod
    def forward(ctx, local, group=None):
        import torch.distributed as dist
        ctx.group = group
        world = dist.get_world_size(group)
        out = torch.empty((world * local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(out, local.contiguous(), group=group)
        return out

    @staticmethod
    def backward(ctx, grad):
        import torch.distributed as dist
        world = dist.get_world_size(ctx.group)
        grad = grad.contiguous()
        out = torch.empty((grad.shape[0] // world,) + tuple(grad.shape[1:]), dtype=grad.dtype, device=grad.device)
        if dist.get_backend(ctx.group) == "nccl":
            dist.reduce_scatter_tensor(out, grad, group=ctx.group)
        else:   # gloo (CPU tests) has no reduce-scatter: sum everything, keep this rank's chunk
            full = grad.clone()
            dist.all_reduce(full, group=ctx.group)
            out.copy_(full.view(world, *out.shape)[dist.get_rank(ctx.group)])
        return out, None


def dist_all_gather(local: torch.Tensor, group=None) -> torch.Tensor:
    return DistAllGatherFunction.apply(local, group)


class PhantomLinearFunction(torch.autograd.Function):
    """y = act(L y_prev + sum_{i != rank} D_i g_i + b), g = C y_prev all-gathered (a3);
    backward a7 + a8 + a9.  Shapes follow the reference: y_prev, y are (n/p, batch)."""

    @staticmethod
    def forward(ctx, y_prev, master, layer, comm, rank, activation, layer_index):
        if master is not layer.master:
            raise ConfigurationError("pass the layer's own flat master tensor as the parameter")
        act = as_activation(activation)
        tape = []
        y = pp_forward_layer(layer, y_prev.detach(), comm, rank, tape, activation=act, layer_index=layer_index)
        ctx.layer, ctx.comm, ctx.rank, ctx.act, ctx.layer_index = layer, comm, rank, act, layer_index
        ctx.tape = tape[0]
        ctx.in_dtype = y_prev.dtype
        return y.to(y_prev.dtype) if y.dtype != y_prev.dtype else y

    @staticmethod
    def backward(ctx, grad_y):
        layer, tape, act = ctx.layer, ctx.tape, ctx.act
        dt = layer.dtype
        # delta = dL/dy * act'(preact): ReLU' as a mask kernel over the native [batch, s] buffer
        d = _native(grad_y, dt).contiguous()
        if act is Activation.RELU:
            pre = tape._pre
            kernels.ctx_for(d).call("ppx_relu_mask", kernels.ppx_dtype(dt), d.shape[0], d.shape[1], d.data_ptr(),
                                    kernels.ld(d), pre.data_ptr(), kernels.ld(pre), kernels.stream_handle())
        delta = d.t()
        r = pp_exchange_error_phantoms(layer, delta, ctx.comm, ctx.rank, layer_index=ctx.layer_index)
        grads = pp_param_grads(layer, delta, tape, r)
        grad_in = None
        if ctx.needs_input_grad[0]:
            grad_in = pp_backward_layer(layer, delta, None, Activation.IDENTITY, ctx.comm, ctx.rank,
                                        layer_index=ctx.layer_index, received=r)
            grad_in = grad_in.to(ctx.in_dtype)
        return grad_in, grads.flat, None, None, None, None, None


def phantom_linear(y_prev: torch.Tensor, layer: PhantomLayer, comm, rank: int, activation=Activation.RELU,
                   layer_index: int = 0) -> torch.Tensor:
    """Autograd-aware phantom layer; `layer.master` must be a leaf with requires_grad=True to
    receive the flat gradient."""
    return PhantomLinearFunction.apply(y_prev, layer.master, layer, comm, rank, activation, layer_index)

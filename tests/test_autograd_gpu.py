"""PhantomLinearFunction (forward a3, backward a7+a8+a9) through torch.autograd, one rank per
thread over the in-process Communicator, against the reference's golden gradients (fp32 tier,
1e-4 normwise, tests/golden/tiny.npz produced by phantomsim itself)."""


import pytest
import torch

from test_phantom_gpu import _model_np, _tiny, nerr

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("ci", [3, 5, 6])     # ReLU stacks (p = 4), sum and mean losses
def test_autograd_layers_match_reference_gradients(ci):
    from paper_2508_00960_b200.autograd import phantom_linear
    from paper_2508_00960_b200.collectives import Communicator
    from paper_2508_00960_b200.phantom import grads_from_flat, model_from_numpy
    z = _tiny()
    pre = f"c{ci}_"
    n, p, k, L, B, seed = (int(v) for v in z[pre + "cfg"])
    act, red = str(z[pre + "act"]), str(z[pre + "red"])
    s = n // p
    model = model_from_numpy(_model_np(z, pre, p, L, s), n, p, k, [act] * L, dtype=torch.float32)
    for row in model.rank_layers:
        for lay in row:
            lay.master.requires_grad_(True)
    x = torch.from_numpy(z[pre + "x"]).cuda().float()
    y = torch.from_numpy(z[pre + "y"]).cuda().float()
    comm = Communicator(p)

    def rank(c, r):
        out = x[r * s:(r + 1) * s]
        with torch.autograd.set_multithreading_enabled(False):
            for l in range(L):
                out = phantom_linear(out, model.rank_layers[r][l], c, r, model.activations[l], layer_index=l)
            diff = out - y[r * s:(r + 1) * s]
            loss = 0.5 * (diff * diff).sum()
            if red == "mean":
                loss = loss / B
            loss.backward()
        return out.detach()

    outs = comm.run(rank)
    torch.cuda.synchronize()
    for r in range(p):
        assert nerr(outs[r], z[f"{pre}r{r}_y_out"]) <= 1e-4
        for l in range(L):
            q = f"{pre}r{r}_l{l}_"
            g = grads_from_flat(model.rank_layers[r][l].master.grad, s, k, p, r)
            assert nerr(g.local, z[q + "g_local"]) <= 1e-4, (r, l, "local")
            assert nerr(g.compressor, z[q + "g_comp"]) <= 1e-4, (r, l, "comp")
            assert nerr(g.bias, z[q + "g_bias"]) <= 1e-4, (r, l, "bias")
            dec = torch.stack([g.decompressors[i] for i in sorted(g.decompressors)])
            assert nerr(dec, z[q + "g_dec"]) <= 1e-4, (r, l, "dec")
    # one all-gather per layer forward and one reduce-scatter per layer backward (Table I)
    kinds = [rec.collective.value for rec in comm.records]
    assert kinds.count("all_gather") == L and kinds.count("reduce_scatter") == L

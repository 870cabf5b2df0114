"""Generate the PSHARD01 golden checkpoints with the UNMODIFIED reference (phantomsim.checkpoint).

Weights are rounded to fp32 precision first (still stored as float64 by the reference), so a
B200 model whose master weights are fp32 must reproduce these files byte for byte.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_checkpoint_golden.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _round32(a):
    a[...] = np.asarray(a, dtype=np.float32).astype(np.float64)


def main():
    sys.path.insert(0, REF_SRC)
    import phantomsim as ps
    from phantomsim.checkpoint import load_model, save_model

    R, I = ps.Activation.RELU, ps.Activation.IDENTITY
    arrays = {}
    # phantom, all ReLU (loads into the engine), nonzero biases
    pp = ps.init_phantom_model(16, 4, 2, 2, R, seed=3)
    rng = np.random.default_rng(7)
    for j, row in enumerate(pp.rank_layers):
        for l, lay in enumerate(row):
            lay.bias[...] = rng.standard_normal(lay.bias.shape)
            for a in [lay.local, lay.compressor, lay.bias] + [lay.decompressors[i] for i in sorted(lay.decompressors)]:
                _round32(a)
    save_model(os.path.join(HERE, "pp_small.pshard"), pp)
    back = load_model(os.path.join(HERE, "pp_small.pshard"))
    for j, row in enumerate(back.rank_layers):
        for l, lay in enumerate(row):
            arrays[f"pp_{j}_{l}_local"] = lay.local
            arrays[f"pp_{j}_{l}_compressor"] = lay.compressor
            for i in sorted(lay.decompressors):
                arrays[f"pp_{j}_{l}_dec{i}"] = lay.decompressors[i]
            arrays[f"pp_{j}_{l}_bias"] = lay.bias
    # phantom with mixed activations and an odd k
    mix = ps.init_phantom_model(24, 3, 3, 3, [R, I, R], seed=11)
    for row in mix.rank_layers:
        for lay in row:
            for a in [lay.local, lay.compressor, lay.bias] + [lay.decompressors[i] for i in sorted(lay.decompressors)]:
                _round32(a)
    save_model(os.path.join(HERE, "pp_mixed.pshard"), mix)
    # tensor-parallel
    tp = ps.init_tp_model(16, 4, 2, R, seed=5)
    for row in tp.rank_layers:
        for lay in row:
            _round32(lay.weight)
            _round32(lay.bias)
    save_model(os.path.join(HERE, "tp_small.pshard"), tp)
    back = load_model(os.path.join(HERE, "tp_small.pshard"))
    for j, row in enumerate(back.rank_layers):
        for l, lay in enumerate(row):
            arrays[f"tp_{j}_{l}_weight"] = lay.weight
            arrays[f"tp_{j}_{l}_bias"] = lay.bias
    np.savez_compressed(os.path.join(HERE, "checkpoints.npz"), **arrays)
    print("wrote pp_small.pshard, pp_mixed.pshard, tp_small.pshard, checkpoints.npz")


if __name__ == "__main__":
    main()

"""PSHARD01 format (reference checkpoint.py) on the host: the golden files written by the
unmodified reference (tests/golden/make_checkpoint_golden.py) parse to the reference's arrays and
are re-emitted byte for byte; malformed files raise ConfigurationError like the reference."""
import os

import numpy as np
import pytest

from paper_2508_00960_b200 import checkpoint as ck
from paper_2508_00960_b200.errors import ConfigurationError

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
ARR = np.load(os.path.join(GOLD, "checkpoints.npz"))


def _path(name):
    return os.path.join(GOLD, name)


def test_phantom_golden_parses_to_reference_arrays():
    mode, n, p, k, layers, seed, acts = ck.read_header(_path("pp_small.pshard"))
    assert (mode, n, p, k, layers, seed) == (0, 16, 4, 2, 2, 3)
    geo = ck.Geometry(mode, n, p, k, layers)
    ck.check_size(_path("pp_small.pshard"), geo)
    for j in range(p):
        for l in range(layers):
            mats = ck.read_block(_path("pp_small.pshard"), geo, j, l)
            assert np.array_equal(mats[0], ARR[f"pp_{j}_{l}_local"])
            assert np.array_equal(mats[1], ARR[f"pp_{j}_{l}_compressor"])
            peers = [i for i in range(p) if i != j]
            for q, i in enumerate(peers):
                assert np.array_equal(mats[2 + q], ARR[f"pp_{j}_{l}_dec{i}"])
            assert np.array_equal(mats[-1], ARR[f"pp_{j}_{l}_bias"])


def test_tensor_golden_parses_to_reference_arrays():
    mode, n, p, k, layers, seed, acts = ck.read_header(_path("tp_small.pshard"))
    assert (mode, n, p, k, layers, seed) == (1, 16, 4, 0, 2, 5)
    geo = ck.Geometry(mode, n, p, k, layers)
    for j in range(p):
        for l in range(layers):
            w, b = ck.read_block(_path("tp_small.pshard"), geo, j, l)
            assert np.array_equal(w, ARR[f"tp_{j}_{l}_weight"]) and np.array_equal(b, ARR[f"tp_{j}_{l}_bias"])


@pytest.mark.parametrize("name", ["pp_small.pshard", "pp_mixed.pshard", "tp_small.pshard"])
def test_host_rewrite_is_byte_identical(tmp_path, name):
    src = _path(name)
    mode, n, p, k, layers, seed, acts = ck.read_header(src)
    geo = ck.Geometry(mode, n, p, k, layers)
    out = tmp_path / name
    with open(out, "wb") as fh:
        fh.write(ck._header_bytes(mode, n, p, k, layers, seed, acts))
        for j in range(p):
            for l in range(layers):
                ck.write_block(fh, geo, j, l, ck.read_block(src, geo, j, l))
    assert out.read_bytes() == open(src, "rb").read()


def test_block_offsets_tile_the_file():
    geo = ck.Geometry(0, 24, 3, 3, 3)
    assert geo.block_offset(0, 0) == geo.data_start
    assert geo.block_offset(2, 2) + 8 * geo.block_elems == geo.file_size == os.path.getsize(_path("pp_mixed.pshard"))


@pytest.mark.parametrize("mutate, msg", [
    (lambda b: b"XSHARD01" + b[8:], "bad magic"),
    (lambda b: b[:20], "short header"),
    (lambda b: b[:8] + b"\x07" + b[9:], "unknown mode byte"),
    (lambda b: b[:ck._HEADER.size] + b"\x05" + b[ck._HEADER.size + 1:], "unknown activation code"),
])
def test_malformed_headers(tmp_path, mutate, msg):
    raw = open(_path("pp_small.pshard"), "rb").read()
    bad = tmp_path / "bad.pshard"
    bad.write_bytes(mutate(raw))
    with pytest.raises(ConfigurationError, match=msg):
        ck.read_header(bad)


@pytest.mark.parametrize("delta, msg", [(-8, "truncated"), (8, "trailing bytes")])
def test_size_errors(tmp_path, delta, msg):
    raw = open(_path("pp_small.pshard"), "rb").read()
    bad = tmp_path / "bad.pshard"
    bad.write_bytes(raw[:delta] if delta < 0 else raw + b"\0" * delta)
    geo = ck.Geometry(*ck.read_header(bad)[:5])
    with pytest.raises(ConfigurationError, match=msg):
        ck.check_size(bad, geo)

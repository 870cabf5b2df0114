"""CPU-side checks of the drop-in boundary: libppx.so loads, exports every entry point declared in
include/ppx.h, agrees with the Python flat-layout arithmetic, and refuses CPU tensors (there is
no CPU fallback anywhere in the product path)."""
import os
import re
import subprocess

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2508_00960_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        subprocess.run(["bash", os.path.join(ROOT, "build.sh")], check=True)
    return _lib.load()


def header_functions():
    src = open(os.path.join(ROOT, "include", "ppx.h")).read()
    return sorted(set(re.findall(r"^\s*(?:ppx_status|int|int32_t|int64_t|const char\*)\s+(ppx_\w+)\s*\(", src, re.M)))


def test_every_declared_symbol_is_exported(lib):
    names = header_functions()
    assert len(names) >= 25
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_header(lib):
    from paper_2508_00960_b200 import _lib
    assert set(header_functions()) <= set(_lib.EXPORTS)


def test_abi_version_and_layout(lib):
    from paper_2508_00960_b200.core import flat_offsets
    assert lib.ppx_abi_version() == 1
    for s, k, p in [(2048, 128, 8), (512, 16, 2), (2, 1, 2), (4096, 64, 4), (16, 3, 1)]:
        assert lib.ppx_layer_elems(s, k, p) == flat_offsets(s, k, p)["total"]
    # with s, k multiples of 8 the flat block is exactly the PSHARD01 record (checkpoint.py:57-64)
    s, k, p = 2048, 128, 8
    assert flat_offsets(s, k, p)["total"] == s * s + k * s + (p - 1) * s * k + s


def test_bad_arguments_map_to_configuration_error(lib):
    from paper_2508_00960_b200 import _lib
    from paper_2508_00960_b200.errors import ConfigurationError
    assert lib.ppx_create(0, 0, 0, None, None) == _lib.PPX_E_CONFIG
    with pytest.raises(ConfigurationError):
        _lib.check(_lib.PPX_E_CONFIG, None, "x")


def test_cpu_tensors_are_refused():
    from paper_2508_00960_b200 import kernels
    from paper_2508_00960_b200.errors import ConfigurationError
    with pytest.raises(ConfigurationError):
        kernels.ptr(torch.zeros(4))


def test_phantom_layer_validation_matches_reference():
    """phantom.py:32-46 shape checks run before any device work."""
    from paper_2508_00960_b200.errors import ConfigurationError
    from paper_2508_00960_b200.phantom import PhantomLayer
    with pytest.raises(ConfigurationError):
        PhantomLayer(np.ones((2, 3)), np.ones((1, 2)), {}, np.zeros(2), device="cpu")
    with pytest.raises(ConfigurationError):
        PhantomLayer(np.ones((2, 2)), np.ones((3, 2)), {}, np.zeros(2), device="cpu")


def test_sizing_functions():
    from paper_2508_00960_b200.phantom import pp_model_size, valid_k
    assert pp_model_size(16384, 8, 16, 2) == 71_303_168
    assert pp_model_size(4, 2, 1, 1) == 4 * 4 // 2 + 2 * 1 * 4
    assert valid_k(16384, 8) == (2048, 1792.0)

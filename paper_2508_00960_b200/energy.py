"""Measured energy (NVML total-energy counter, reference energy.py's modeled J replaced by the
device's own meter): joules consumed by one GPU between two reads.

NVML numbers GPUs in PCI order and ignores CUDA_VISIBLE_DEVICES / CUDA_DEVICE_ORDER, so the
handle of CUDA device i is looked up by the device's UUID (nvml_handle), never by ordinal."""

from __future__ import annotations

_nvml = None
_handles: dict = {}


def _init():
    global _nvml
    if _nvml is None:
        import pynvml
        pynvml.nvmlInit()
        _nvml = pynvml
    return _nvml


def nvml_handle(cuda_index: int):
    """NVML handle of CUDA device `cuda_index` (by UUID; PCI bus id, then ordinal as fallbacks)."""
    if cuda_index in _handles:
        return _handles[cuda_index]
    nv = _init()
    h = None
    try:
        import torch
        props = torch.cuda.get_device_properties(cuda_index)
        uuid = str(getattr(props, "uuid", "") or "")
        if uuid:
            uuid = uuid if uuid.startswith("GPU-") else "GPU-" + uuid
            h = nv.nvmlDeviceGetHandleByUUID(uuid)
    except Exception:
        h = None
    if h is None:
        try:
            import torch
            props = torch.cuda.get_device_properties(cuda_index)
            bus = f"{getattr(props, 'pci_domain_id', 0):08x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
            h = nv.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            h = None
    if h is None:
        h = nv.nvmlDeviceGetHandleByIndex(cuda_index)
    _handles[cuda_index] = h
    return h


def energy_mj(gpu_index: int) -> float | None:
    """Cumulative energy of CUDA device `gpu_index` in millijoules (None when NVML is unavailable)."""
    try:
        return float(_init().nvmlDeviceGetTotalEnergyConsumption(nvml_handle(gpu_index)))
    except Exception:
        return None


class EnergyMeter:
    """with EnergyMeter(dev) as m: ... ; m.joules (None without NVML, or when the window was shorter
    than `min_seconds`: the total-energy counter advances in coarse steps, so sub-second windows
    read 0 or one whole step)."""

    def __init__(self, gpu_index: int, min_seconds: float = 1.0):
        self.gpu, self.joules, self.min_seconds = gpu_index, None, min_seconds

    def __enter__(self):
        import time
        self._t0 = time.perf_counter()
        self._e0 = energy_mj(self.gpu)
        return self

    def __exit__(self, *exc):
        import time
        e1 = energy_mj(self.gpu)
        self.seconds = time.perf_counter() - self._t0
        if self._e0 is not None and e1 is not None and self.seconds >= self.min_seconds:
            self.joules = (e1 - self._e0) / 1e3
        return False

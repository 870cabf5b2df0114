"""Measured energy (NVML total-energy counter, reference energy.py's modeled J replaced by the
device's own meter): joules consumed by one GPU between two reads."""

from __future__ import annotations

_nvml = None


def energy_mj(gpu_index: int) -> float | None:
    """Cumulative energy of GPU `gpu_index` in millijoules (None when NVML is unavailable)."""
    global _nvml
    try:
        if _nvml is None:
            import pynvml
            pynvml.nvmlInit()
            _nvml = pynvml
        h = _nvml.nvmlDeviceGetHandleByIndex(gpu_index)
        return float(_nvml.nvmlDeviceGetTotalEnergyConsumption(h))
    except Exception:
        return None


class EnergyMeter:
    """with EnergyMeter(dev) as m: ... ; m.joules (None without NVML)."""

    def __init__(self, gpu_index: int):
        self.gpu, self.joules = gpu_index, None

    def __enter__(self):
        self._e0 = energy_mj(self.gpu)
        return self

    def __exit__(self, *exc):
        e1 = energy_mj(self.gpu)
        if self._e0 is not None and e1 is not None:
            self.joules = (e1 - self._e0) / 1e3
        return False

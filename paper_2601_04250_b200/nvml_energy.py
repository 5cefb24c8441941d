"""Real energy signal from NVML, telemetry only.

The reference's E(x) comes from simulated joules fed to the `EnergyLedger`
(energy.py:75-101; servesim.py:303-305, 343, 389).  On a B200 the driver keeps
a total-energy counter per GPU (`nvmlDeviceGetTotalEnergyConsumption`, mJ since
driver load); deltas of it over a window of serving work give measured joules
per admitted inference, which the ledger's own kWh / CO2 arithmetic
(`energy.to_kwh`, `energy.co2_of`) turns into the paper's reporting units.  Not
fed back into the controller yet (telemetry first, as §8f ranks it); the
counter's update period (tens of ms) makes windows shorter than ~0.2 s noisy.
"""

from __future__ import annotations

from .energy import DEFAULT_GRID_INTENSITY, co2_of, to_kwh


class NvmlUnavailable(RuntimeError):
    """NVML (nvidia-ml-py / the driver) is not usable on this host."""


class NvmlEnergyMeter:
    """Joules consumed by one GPU between `start()` and `stop()`."""

    def __init__(self, index: int = 0) -> None:
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(int(index))
            pynvml.nvmlDeviceGetTotalEnergyConsumption(self._h)
        except Exception as exc:   # no driver / no GPU / counter unsupported
            raise NvmlUnavailable(f"NVML energy counter unavailable: {exc}") from None
        self._t0: int | None = None

    @classmethod
    def for_cuda_device(cls, device: int) -> "NvmlEnergyMeter":
        """The meter of CUDA device `device`, matched by PCI address (CUDA's device
        order need not be NVML's); falls back to the same index."""
        m = cls.__new__(cls)
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            pr = torch.cuda.get_device_properties(device)
            bus = f"{pr.pci_domain_id:08X}:{pr.pci_bus_id:02X}:{pr.pci_device_id:02X}.0"
            m._nvml = pynvml
            m._h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            pynvml.nvmlDeviceGetTotalEnergyConsumption(m._h)
            m._t0 = None
            return m
        except Exception:
            return cls(device)

    def read_mj(self) -> int:
        return int(self._nvml.nvmlDeviceGetTotalEnergyConsumption(self._h))

    def start(self) -> None:
        self._t0 = self.read_mj()

    def stop(self) -> float:
        """Joules since `start()`."""
        if self._t0 is None:
            raise RuntimeError("stop() before start()")
        j = (self.read_mj() - self._t0) / 1000.0
        self._t0 = None
        return j


def energy_report(joules: float, inferences: float,
                  grid_intensity: float = DEFAULT_GRID_INTENSITY) -> dict:
    """Joules per inference and the ledger's units per million inferences."""
    per = joules / inferences if inferences > 0 else float("nan")
    kwh_per_m = to_kwh(per * 1e6) if per == per and per >= 0 else float("nan")
    return {"joules": joules, "inferences": inferences, "joules_per_inference": per,
            "kwh_per_million": kwh_per_m,
            "kg_co2_per_million": co2_of(kwh_per_m, grid_intensity) if kwh_per_m == kwh_per_m else float("nan"),
            "grid_intensity_kg_per_kwh": grid_intensity}

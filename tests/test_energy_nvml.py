"""NVML energy telemetry (paper_2601_04250_b200.nvml_energy)."""

from __future__ import annotations

import math

import pytest


def test_energy_report_units():
    from paper_2601_04250_b200.energy import co2_of, to_kwh
    from paper_2601_04250_b200.nvml_energy import energy_report
    r = energy_report(360.0, 1000.0, grid_intensity=0.4)
    assert r["joules_per_inference"] == 0.36
    assert r["kwh_per_million"] == to_kwh(0.36 * 1e6) == 0.1
    assert r["kg_co2_per_million"] == co2_of(0.1, 0.4)
    assert math.isnan(energy_report(1.0, 0.0)["joules_per_inference"])


def test_meter_fails_loudly_without_nvml():
    import torch
    from paper_2601_04250_b200.nvml_energy import NvmlEnergyMeter, NvmlUnavailable
    if torch.cuda.is_available():
        pytest.skip("GPU host: covered by the gpu test")
    with pytest.raises(NvmlUnavailable):
        NvmlEnergyMeter(0)


@pytest.mark.gpu
def test_meter_measures_gpu_work():
    import time
    import torch
    from paper_2601_04250_b200.nvml_energy import NvmlEnergyMeter
    m = NvmlEnergyMeter(torch.cuda.current_device())
    a = torch.randn((8192, 8192), device="cuda", dtype=torch.bfloat16)
    m.start()
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 0.5:
        for _ in range(20):
            a = (a @ a).clamp_(-1, 1)
        torch.cuda.synchronize()
    j = m.stop()
    secs = time.perf_counter() - t0
    assert j > 0.0 and 50.0 < j / secs < 2000.0, (j, secs)   # a B200 under load: 50 W .. 2 kW

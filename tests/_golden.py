"""Loaders for the committed golden fixtures (tests/golden/, made by make_golden.py)."""

from __future__ import annotations

import json
import os

import numpy as np

from paper_2601_04250_b200 import _abi

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

SIM_NAMES = ["demo03", "demo03_all_channels", "ablation", "energy_sweep", "onoff_bursty", "lt_omc"]
REPLAY_NAMES = ["k2_ablation", "k1000_softmax", "k4_lt_omc"]


def kat() -> dict:
    with open(os.path.join(GOLDEN, "kat.json")) as f:
        return json.load(f)


def npz(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, name + ".npz"), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def rows_from_base(base: np.ndarray) -> np.ndarray:
    """Same recipe as make_golden.rows_from_base (exact integer arithmetic)."""
    num = base.astype(np.int64) ** 4
    den = num.sum(axis=1, keepdims=True)
    return num.astype(np.float64) / den.astype(np.float64)


def replay(name: str) -> dict:
    d = npz("replay_" + name)
    if "rows_base" in d:
        rows = rows_from_base(d["rows_base"])
        r, c, v = d["patch"]
        rows[int(r), int(c)] = v
        d["rows"] = rows
    d["params"] = json.loads(str(d["params"]))
    d["final_state"] = json.loads(str(d["final_state"]))
    return d


def sim(name: str) -> dict:
    d = npz("sim_" + name)
    d["params"] = json.loads(str(d["params"]))
    d["final_state"] = json.loads(str(d["final_state"]))
    return d


def abi_params(p: dict) -> _abi.gg_params:
    return _abi.gg_params(p["alpha"], p["beta"], p["gamma"], p["tau0"], p["tau_inf"], p["k"],
                          p["ewma_lambda"], p["direction"], p["utility_proxy"], p["routing"],
                          p["queue_threshold"], p["p95_window"], 0)


def state_dict_of_abi(s: _abi.gg_state) -> dict:
    def ch(c):
        return [c.lo, c.hi] if c.seen else None
    return dict(energy=ch(s.n_energy), queue_depth=ch(s.n_queue_depth), p95_ms=ch(s.n_p95_ms),
                ewma=s.ewma_joules_per_request, samples_seen=s.samples_seen,
                total_joules=s.total_joules, admitted_total=s.admitted_total,
                skipped_total=s.skipped_total, p95_current=s.p95_current, t_origin=s.t_origin)

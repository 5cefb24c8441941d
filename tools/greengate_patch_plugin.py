"""pytest plugin: run the reference's own test suite with the device controller patched in.

    PYTHONPATH=baseline/_ref:<repo>:<repo>/tools \
        python -m pytest -p greengate_patch_plugin baseline/_ref/greengate_suite/tests

`patch_greengate` (paper_2601_04250_b200/integration.py) routes every
`ControllerConfig.build(...)` of the reference — Simulation.__init__
(servesim.py:185-190), GatewayState.__init__ (gateway.py:51-56), the tests'
own `config.build(EnergyLedger())` — to the sm_100a AdmissionController.  At
session end the number of device controllers built is written to
$GG_PATCH_REPORT (JSON) so the caller can prove the patch was active.
"""

import json
import os

import greengate

from paper_2601_04250_b200 import controller as _dev
from paper_2601_04250_b200.integration import patch_greengate

_BUILT = {"device_controllers": 0, "decide_calls": 0, "outcome_calls": 0}
_orig_init = _dev.AdmissionController.__init__
_orig_decide = _dev.AdmissionController.decide
_orig_outcome = _dev.AdmissionController.record_outcome


def _init(self, *a, **kw):
    _BUILT["device_controllers"] += 1
    _orig_init(self, *a, **kw)


def _decide(self, *a, **kw):
    _BUILT["decide_calls"] += 1
    return _orig_decide(self, *a, **kw)


def _outcome(self, *a, **kw):
    _BUILT["outcome_calls"] += 1
    return _orig_outcome(self, *a, **kw)


_dev.AdmissionController.__init__ = _init
_dev.AdmissionController.decide = _decide
_dev.AdmissionController.record_outcome = _outcome
patch_greengate(greengate)


def pytest_sessionfinish(session, exitstatus):
    path = os.environ.get("GG_PATCH_REPORT")
    if path:
        with open(path, "w") as f:
            json.dump(dict(_BUILT, greengate=greengate.__file__), f)

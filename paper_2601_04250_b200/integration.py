"""Drop-in wiring into an installed reference `greengate` package.

    import greengate
    from paper_2601_04250_b200.integration import patch_greengate
    patch_greengate(greengate)          # every ControllerConfig.build now returns the
                                        # device-backed AdmissionController

After the patch the reference's own call sites — Simulation.__init__
(servesim.py:185-190), GatewayState.__init__ (gateway.py:51-56), the CLI and
the demos — construct the B200 controller through their unchanged
`config.controller.build(ledger, congestion_source, p95_window=..., t_origin=...)`
call; decide()/record_outcome()/p95_ms()/reset_clock() and the counters are
served by the sm_100a kernels.  The reference's EnergyLedger passed in is
mirrored (its ewma/samples/total fields are refreshed after every outcome), so
RunTrace.ledger and /v1/state keep reporting the loop state.
"""

from __future__ import annotations

from . import controller as _dev
from . import errors as _errors


def _device_build(self, ledger=None, congestion_source=None, *, p95_window: int = 100,
                  t_origin: float = 0.0):
    cfg = _dev.ControllerConfig(
        enabled=self.enabled, alpha=self.alpha, beta=self.beta, gamma=self.gamma,
        tau0=self.tau0, tau_inf=self.tau_inf, k=self.k,
        direction=_dev.Direction[self.direction.name],
        utility_proxy=_dev.UtilityProxy[self.utility_proxy.name],
        routing=_dev.RoutePolicy[self.routing.name], queue_threshold=self.queue_threshold)
    if ledger is None:
        from .energy import EnergyLedger
        ledger = EnergyLedger()
    ctl = cfg.build(ledger, congestion_source, p95_window=p95_window, t_origin=t_origin)
    # decide() returns the host package's own AdmissionDecision/ServicePath/Reason
    # members, so identity checks like `path is ServicePath.DIRECT` keep working
    import sys
    host_mod = sys.modules[type(self).__module__]
    ctl.result_types = host_mod
    # ... and raises exceptions the host's handlers catch: gateway.py:199/228
    # (`except InvalidDistribution` / `except NegativeMeasurement` -> HTTP 400),
    # cli.py:202 (`except GreengateError`)
    host_pkg = host_mod.__name__.rpartition(".")[0]
    host_errors = sys.modules.get(host_pkg + ".errors") if host_pkg else None
    if host_errors is not None:
        ctl.errors = _bridged_errors(host_errors)
    return ctl


_BRIDGED: dict = {}


def _bridged_errors(host_errors):
    """Namespace of exception classes that derive from both the host package's
    class and ours of the same name (cached per host module)."""
    key = id(host_errors)
    ns = _BRIDGED.get(key)
    if ns is None:
        import types
        ns = types.SimpleNamespace()
        for name in ("InvalidDistribution", "NegativeMeasurement", "InvalidSchedule",
                     "InvalidLambda"):
            ours, theirs = getattr(_errors, name), getattr(host_errors, name, None)
            cls = ours if theirs is None else type(name, (theirs, ours), {
                "__module__": host_errors.__name__, "__doc__": theirs.__doc__})
            setattr(ns, name, cls)
        _BRIDGED[key] = ns
    return ns


def patch_greengate(greengate_module) -> None:
    """Route the reference ControllerConfig.build (controller.py:235-253) to the device."""
    cc = greengate_module.controller.ControllerConfig
    if getattr(cc, "_b200_patched", False):
        return
    cc._reference_build = cc.build
    cc.build = _device_build
    cc._b200_patched = True


def unpatch_greengate(greengate_module) -> None:
    cc = greengate_module.controller.ControllerConfig
    if getattr(cc, "_b200_patched", False):
        cc.build = cc._reference_build
        cc._b200_patched = False

"""B200-native (sm_100a) gated-inference hot path of arXiv 2601.04250 ("Green MLOps").

Drop-in for the reference `greengate` controller API (pkg/src/greengate):
the admission step (K1), outcome feedback (K2) and logit epilogue (K3) run as
hand-written CUDA kernels behind the C ABI in include/greengate_b200.h; the
admitted batch runs a hand-written DistilBERT / ResNet-18 forward.  There is
no CPU fallback.
"""

from .controller import (
    AdmissionController,
    AdmissionDecision,
    BatchDecision,
    CongestionSnapshot,
    ControllerConfig,
    CostBreakdown,
    CostWeights,
    Direction,
    NormalizerChannel,
    NormalizerState,
    Reason,
    RoutePolicy,
    ServicePath,
    ThresholdSchedule,
    UtilityProxy,
    cost,
    entropy_utility,
    one_minus_confidence_utility,
    threshold_at,
)
from .energy import EnergyLedger, co2_of, ewma_update, to_kwh
from .errors import (
    ConfigError,
    EmptyTrace,
    GreengateError,
    InvalidDistribution,
    InvalidLambda,
    InvalidSchedule,
    MismatchedRun,
    NegativeMeasurement,
)
from .workload import (
    ArrivalMode,
    RequestFeatures,
    Trace,
    WorkloadConfig,
    generate_requests,
    generate_trace,
    onoff_arrivals,
    onoff_phases,
    poisson_arrivals,
    synth_request,
)

__version__ = "0.1.0"

"""B200-native MoE-offloading decode engine (hot path of arXiv 2511.05814).

Drop-in modules mirroring the reference simulator's API (moesim/__init__.py:11-61):
traces, policies, kernels, simulate, toymoe, metrics, costmodel, errors.  The compute
behind them is libmoeb200.so (CUDA, sm_100a) reached through the C ABI in
include/moeb200.h; `engine.OffloadEngine` is the Mixtral-shaped offload decode engine.
"""

from .errors import ConfigError, MoesimError, TraceError, TraceParseError, TraceValidationError
from .policies import CacheState, PolicyKind, StepOutcome, policy_step, warm_state
from .traces import (
    ActivationRecord,
    ActivationTrace,
    ExpertId,
    ModelShape,
    SpeculationRecord,
    SpeculationTrace,
    load_trace,
    read_trace,
    save_trace,
    write_trace,
)
from .simulate import (
    CacheEventLog,
    SimConfig,
    load_event_log,
    offloads_to_cache_size,
    save_event_log,
    simulate,
)
from .metrics import CacheMetrics, SpeculationMetrics, cache_metrics, speculation_metrics
from .costmodel import CostParams, estimate_latency, speculation_cost
from .toymoe import (
    GatingNetwork,
    HiddenState,
    ToyModelConfig,
    ToyMoeModel,
    forward_token,
    gate_select,
    run_model,
    speculate_next,
)
from .tracegen import MarkovParams, ZipfParams, gen_markov, gen_zipf, repeat_rate
from .engine import EngineConfig, OffloadEngine

__version__ = "0.1.0"

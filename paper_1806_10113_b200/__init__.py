"""offsim-b200: the B200 (sm_100a) hot path of arXiv 1806.10113's temporal
execution model, behind the reference package's API (offsim).

Drop-in names (same signatures and semantics as /root/reference's
offsim/__init__.py:3-55 for the hot path):
    simulate, exhaustive_search, reorder_batch, select_first_task,
    select_next_task, select_last_tasks, recompute_overlap, make_report,
    DeviceProfile, TaskSpec, Command, Timeline, PermutationReport,
    stage_times, estimate_transfer, estimate_kernel, fit_kernel_model,
    classify_task
Batched / summary-mode additions (no reference equivalent; the reference
only loops in Python):
    exhaustive_summary, exhaustive_summary_batch, reorder_batch_many,
    reorder_durs
Every simulation runs in liboffsim_b200.so; importing the package does not
load it, the first call does, and fails loudly if it is missing.
"""

from .engine import KINDS, Command, Timeline, idle_report, recompute_overlap, simulate
from .heuristic import (
    SUM_MODE,
    reorder_batch,
    reorder_batch_many,
    reorder_durs,
    select_first_task,
    select_last_tasks,
    select_next_task,
)
from .model import (
    DeviceProfile,
    Direction,
    InsufficientSamples,
    NegativeFitWarning,
    OffsimError,
    TaskDominance,
    TaskSpec,
    UnresolvableDuration,
    classify_task,
    estimate_kernel,
    estimate_transfer,
    fit_kernel_model,
    stage_times,
)
from .micro import micro_simulate, validate
from .noreorder import noreorder_distribution, simulate_sequence
from .workload import (
    Benchmark,
    Scenario,
    ScenarioResult,
    load_bk_benchmark,
    load_table2_tasks,
    run_scenario,
    sample_real_tasks,
)
from .search import (
    DEFAULT_CAP,
    OrderingStats,
    OrderingSummary,
    PermutationReport,
    exhaustive_search,
    exhaustive_stats,
    exhaustive_stats_durs,
    exhaustive_summary,
    exhaustive_summary_batch,
    exhaustive_summary_durs,
    heuristic_percentile,
    make_report,
    sample_permutations,
)

__version__ = "0.1.0"

__all__ = [
    "Benchmark", "Scenario", "ScenarioResult", "load_bk_benchmark", "load_table2_tasks", "run_scenario",
    "sample_real_tasks",
    "Command", "DeviceProfile", "Direction", "InsufficientSamples", "KINDS", "NegativeFitWarning",
    "OffsimError", "OrderingStats", "OrderingSummary", "PermutationReport", "SUM_MODE", "TaskDominance", "TaskSpec",
    "Timeline", "UnresolvableDuration", "classify_task", "DEFAULT_CAP", "estimate_kernel",
    "estimate_transfer", "exhaustive_search", "exhaustive_summary", "exhaustive_summary_batch",
    "exhaustive_summary_durs", "exhaustive_stats", "exhaustive_stats_durs", "fit_kernel_model",
    "heuristic_percentile", "idle_report", "micro_simulate", "validate", "noreorder_distribution", "simulate_sequence", "make_report", "recompute_overlap",
    "reorder_batch", "reorder_batch_many", "reorder_durs", "sample_permutations", "select_first_task",
    "select_last_tasks", "select_next_task", "simulate", "stage_times",
]

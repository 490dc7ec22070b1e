"""B200-native HALP solver (arXiv 1803.03383), drop-in for lpopt::run_halp.

The numeric work runs in libhalp_b200.so (hand-written sm_100a CUDA kernels
behind the C ABI in include/halp.h); this package is the Python mirror of the
reference's C++ interface (see halp.py) plus the in-tree build (build.py).
"""
from .halp import (  # noqa: F401
    Algorithm, BatchProblems, ClipMode, clipping_variant_config, run_clipping_variant, Dataset, DivergenceError, EpochOption, Error, HalpCudaError, InvalidInputError, LossFamily,
    GridAxis, GridOutcome, GridResult, MetricRow, Objective, OptimizerConfig, RunRecord, UnsupportedError, generate,
    format_double, grid_search, halp_scale, hash_vector, write_run_csv,
    oracle_plan_for, plan_for, resolve_inner_steps, rng_state_after, run, run_halp, run_lp_sgd, run_lp_svrg, run_prepared, run_sgd, run_svrg,
    run_lm_halp, quantize_dataset, data_scale, QuantizedExamples,
    shard_plan,
)
from . import harness  # noqa: F401,E402
from .harness import (  # noqa: F401,E402
    ExperimentSpec, build_dataset, conditioning_sweep, make_conditioned_regression, make_regression, run_experiment,
    write_sweep_csv,
)

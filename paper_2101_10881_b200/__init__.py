"""B200-native evaluation and differentiation of polynomials at truncated
power series in multiple-double precision (arXiv 2101.10881), behind the
reference ``pseval`` API. See pseval.py for the API mirror and
include/pse_b200.h for the C ABI."""
from .pseval import *  # noqa: F401,F403
from .pseval import (CPLX, REAL, DataArray, DevicePlan, JobGraph, Monomial, OpCost, Polynomial, Problem,
                     RunReport, build_jobgraph, build_jobgraph_shape, evaluate, evaluate_packed, flop_count,
                     flop_count_add, flop_count_mul, gen_benchmark, instrumented_cost, md_apply, reporting_cost,
                     run_device, series_add, series_conv, series_scale_int, stage, validate)
from ._lib import InvalidArgument, PseError, LIB_PATH

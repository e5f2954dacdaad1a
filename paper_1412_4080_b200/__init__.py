"""B200-native dynamic-screening sparse solver (hot path of arXiv 1412.4080).

Drop-in for the reference ``screenlab`` solver path: ``run(problem, cfg,
iteration_hook=None) -> SolveResult`` with the same config, result and error
semantics, executed by hand-written sm_100a CUDA kernels in libdynscreen.so
(C ABI: include/dynscreen.h).  Importing the package does not touch the GPU;
the first numerical call loads the library and fails loudly if it or a CUDA
device is missing.
"""

from .instrument import DYNAMIC, NONE, STATIC, STRATEGIES, SolveTrace, flops_iteration, flops_static_init
from .problem import (GROUP, LASSO, Dictionary, GroupPartition, LambdaMax, Problem, expand, group_spectral_norms,
                      index_set, operator_norm, spectral_norm)
from .solver import (ALGORITHMS, CP, DOME, DST3, FISTA, GROUP_TESTS, GSAFE, GST3, ISTA, LASSO_TESTS, SAFE,
                     SPARSA, TWIST, DeviceContext, IterationInfo, ScreenState, SolveResult, SolverConfig, run)
from .ops import (lambda_max, prox_group, prox_l1, screen_update, test_dome, test_sphere_group,
                  test_sphere_lasso)

__version__ = "0.1.0"

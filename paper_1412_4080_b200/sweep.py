"""GPU-resident lambda sweep: the reference's benchmark driver
(cli._bench_seed / run_bench, cli.py:230-292) on the device engine.

The dictionary is uploaded once (cached on the Dictionary object) and every
(lambda ratio, algorithm, strategy, test) run of the grid reuses it; lambda_max is
computed once on the device.  Rows follow the reference's BENCH_HEADER and can be
written in the same CSV format, so the paper's flop_N / flop_S / flop_D figures
(instrument.normalized_metrics) come from the same kernels as the solver.
"""

from __future__ import annotations

import json
import time
from dataclasses import asdict, dataclass, field

from .instrument import NONE, STRATEGIES
from .ops import lambda_max
from .problem import Problem
from .solver import ALGORITHMS, GROUP_TESTS, LASSO_TESTS, SolverConfig, run

BENCH_HEADER = "seed,algo,strategy,test,lambda_ratio,iters,flops,time_s,final_obj,screened_frac"


@dataclass
class SweepPlan:
    """The run grid of one sweep (the grid fields of cli.BenchPlan, cli.py:37-80)."""

    lambda_ratios: list
    algorithms: list = field(default_factory=lambda: ["ista"])
    strategies: list = field(default_factory=lambda: list(STRATEGIES))
    tests: list = field(default_factory=lambda: ["dst3"])
    max_iters: int = 200
    rel_tol: float = 1e-7

    def validate(self, kind):
        ratios = list(self.lambda_ratios)
        if not ratios or ratios != sorted(ratios):
            raise ValueError("lambda ratios must be given in ascending order")
        if ratios[0] <= 0 or ratios[-1] > 1:
            raise ValueError("lambda ratios must lie in (0, 1]")
        allowed = LASSO_TESTS if kind == "lasso" else GROUP_TESTS
        for t in self.tests:
            if t not in allowed:
                raise ValueError(f"test {t!r} not valid for {kind} problems")
        for a in self.algorithms:
            if a not in ALGORITHMS:
                raise ValueError(f"unknown algorithm {a!r}")
        for s in self.strategies:
            if s not in STRATEGIES:
                raise ValueError(f"unknown strategy {s!r}")
        if self.max_iters < 1:
            raise ValueError("max_iters must be positive")


def sweep(dictionary, y, plan, partition=None, seed=0, device_time=False, results=None):
    """Run the grid on one instance; returns BENCH_HEADER rows (cli._bench_seed, cli.py:230-262).

    time_s is host wall time around run() like the reference (device_time=True: the
    device solve time instead).  ``results`` (a list) collects the SolveResult of every row.
    """
    probe = Problem(dictionary, y, 1.0, partition)
    plan.validate(probe.kind)
    lmax = lambda_max(probe).value
    rows = []
    for ratio in plan.lambda_ratios:
        problem = Problem(dictionary, y, ratio * lmax, partition)
        for algo in plan.algorithms:
            for strategy in plan.strategies:
                tests = ["-"] if strategy == NONE else plan.tests
                for test in tests:
                    cfg = SolverConfig(algorithm=algo, strategy=strategy, test=None if test == "-" else test,
                                       max_iters=plan.max_iters, rel_tol=plan.rel_tol)
                    t0 = time.perf_counter()
                    res = run(problem, cfg)
                    elapsed = res.device_seconds if device_time else time.perf_counter() - t0
                    rows.append((seed, algo, strategy, test, ratio, res.iterations, res.trace.total_flops,
                                 elapsed, res.final_objective, res.screened_fraction))
                    if results is not None:
                        results.append(res)
    return rows


def write_bench_csv(rows, path, plan):
    """Same layout as cli.run_bench (cli.py:274-292): config comment, header, sorted rows."""
    rows = sorted(rows, key=lambda r: (r[0], r[1], r[2], r[3], r[4]))
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(f"# paper_1412_4080_b200 sweep config={json.dumps(asdict(plan), sort_keys=True)}\n")
        fh.write(BENCH_HEADER + "\n")
        for row in rows:
            fh.write("{},{},{},{},{!r},{},{},{!r},{!r},{!r}\n".format(*row))
    return len(rows)

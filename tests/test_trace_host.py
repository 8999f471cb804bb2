"""trace_run (sdr.cpp:158-177) host logic, after test_sdr.cpp:146-197, with a
stand-in estimator (no GPU): rows appear every eval_every iterations, carry
the recorded cost and the estimator's own clock, and nothing is traced
without a scorer.  The device runs are in tests/cpp/test_api.cpp."""
import numpy as np

import paper_2605_19388_b200 as dfm


def _fake_fit(iters):
    def run_fit(options):
        costs = 100.0 - np.arange(iters + 1, dtype=float)
        walls = np.full(iters, 0.001)
        if options.eval_every > 0 and options.on_eval:
            for it in range(options.eval_every, iters + 1, options.eval_every):
                options.on_eval(dfm.FitSnapshot(it, float(costs[it]), float(walls[:it].sum()),
                                                dfm.BlockLayout([2]), [], [], np.zeros((1, 1, 2))))
        assert options.floor == 1e-6
        return dfm.FitReport(costs, walls, iters)
    return run_fit


def test_untraced_run_has_no_rows():
    out = dfm.trace_run(_fake_fit(20), None, 0)
    assert out.rows == [] and out.report.iterations == 20


def test_rows_every_eval_every_with_recorded_cost():
    seen = []

    def score(snap):
        seen.append(snap.iteration)
        return 2.5

    out = dfm.trace_run(_fake_fit(20), score, 5)
    assert [r.iteration for r in out.rows] == [5, 10, 15, 20] == seen
    assert all(r.cost == out.report.cost_trace[r.iteration] for r in out.rows)
    assert all(r.mean_sdr_improvement == 2.5 for r in out.rows)
    secs = [r.seconds for r in out.rows]
    assert secs == sorted(secs) and abs(secs[-1] - 0.02) < 1e-12


def test_scorer_without_period_is_not_called():
    out = dfm.trace_run(_fake_fit(8), lambda s: 1 / 0, 0)
    assert out.rows == []

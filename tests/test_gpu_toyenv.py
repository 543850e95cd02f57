"""The toy closed loop (paper_2603_07904_b200/toyenv.py) on the B200 hot
path: the GPU read-out (dyq_qlinear of the feature rows, per-episode widths)
against the oracle's, the GPU dispatcher (dyq_select_bits) bit-exact with the
oracle selector on a recorded trace, and the dynamic-mode suite run end to
end on the GPU reproducing the oracle-driven acceptance properties."""
import numpy as np
import pytest

from paper_2603_07904_b200 import toyenv as T

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from test_gpu_parity import check_close  # noqa: E402
from test_toyenv import HEAD, TOY_THETA, OracleDisp  # noqa: E402

from paper_2603_07904_b200 import dyq  # noqa: E402


@pytest.mark.parametrize("E", [1, 7, 16, 40])
def test_gpu_head_matches_oracle_head(E):
    rng = np.random.default_rng(E)
    s = T.reset(list(range(E)))
    s.phase = rng.integers(0, 4, E)
    s.phase_t = rng.integers(0, 10, E)
    s.d0 = rng.uniform(-0.1, 0.1, (E, 3))
    f = T.features(s)
    head = T.GpuHead()
    for b in ([2] * E, [4] * E, [8] * E, [16] * E, [[2, 4, 8, 16][i % 4] for i in range(E)]):
        b = np.array(b)
        check_close(head(f, b), HEAD(f, b), 1e-3)


def test_gpu_dispatcher_bit_exact_on_a_trace():
    _, _, _, _, tr = T.simulate(list(range(12)), HEAD, T.Static(12, 16))
    acts = np.stack(tr.actions)
    cal = dyq.default_calib(**TOY_THETA)
    g = T.replay_dispatch(acts, T.GpuDispatcher(12, cal))
    o = T.replay_dispatch(acts, OracleDisp(12))
    assert np.array_equal(g, o)
    Mg, Jg = T.kinematic_means(acts, lambda E, lam: T.GpuDispatcher(E, dyq.default_calib(lambda_=lam, **TOY_THETA)))
    Mo, Jo = T.kinematic_means(acts, lambda E, lam: OracleDisp(E, lam=lam))
    assert np.array_equal(Mg, Mo) and np.array_equal(Jg, Jo)


def test_gpu_closed_loop_suite():
    """Dynamic mode with the GPU head and dispatcher over 100 seeds: the
    Pareto property of acceptance 7 holds on the hot path too."""
    seeds = list(range(100))
    head = T.GpuHead()
    cal = dyq.default_calib(**TOY_THETA)
    rep = T.run_suite(seeds, {"static16": lambda E: T.Static(E, 16), "static2": lambda E: T.Static(E, 2),
                              "dynamic": lambda E: T.GpuDispatcher(E, cal)}, head)
    s16, d, s2 = rep["static16"], rep["dynamic"], rep["static2"]
    assert d["success_rate"] >= 0.95 * s16["success_rate"]
    assert d["mean_cost"] <= 0.8 * s16["mean_cost"]
    assert d["success_rate"] >= s2["success_rate"]

"""CUDA-graph replay of a plan (``MpsBatch.capture`` / ``GraphedPlan``): the captured
``reset() + execute(plan)`` gives the eager run's results bit for bit, with the captured
matrices and with new ones of the same circuit structure (a VQE ansatz at new angles)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _state_bits(b):
    import torch
    torch.cuda.synchronize()
    return (b.gamma.cpu().numpy().copy(), b.lam.cpu().numpy().copy(), b.dims.cpu().numpy().copy(),
            b.trunc_err.cpu().numpy().copy(), b.peak.cpu().numpy().copy(), b.mbs.cpu().numpy().copy())


def _assert_same(a, b):
    for x, y in zip(a, b):
        assert x.shape == y.shape and np.array_equal(x, y)


def test_graph_replay_matches_eager_bitwise_and_golden():
    from conftest import load_golden
    from paper_1807_07914_b200 import MpsBatch, TruncationPolicy, compile_batch
    from paper_1807_07914_b200 import workloads as W
    from paper_1807_07914_b200.vqe import batch_energies
    from conftest import assert_scaled_close
    RTOL = 1e-10

    w = W.config2(batch=8)
    w2 = W.config2(seed=77, batch=8)          # same ansatz structure, other angles
    pol = TruncationPolicy(w.cutoff, w.max_bond)
    plan, plan2 = compile_batch(w.programs, w.n), compile_batch(w2.programs, w.n)
    for name in ("items1", "items2", "off1", "off2", "logidx2", "ranges"):
        assert np.array_equal(getattr(plan, name), getattr(plan2, name))

    eager = MpsBatch(8, w.n, pol)
    eager.execute(plan)
    ref1 = _state_bits(eager)
    # cap as the graph's batch will have it (bound model), so the tensors compare shape for shape
    b = MpsBatch(8, w.n, pol, cap=eager.cap)
    gp = b.capture(plan)
    assert b.cap == eager.cap
    _assert_same(_state_bits(b), ref1)        # the recorded run itself
    gp.replay()
    _assert_same(_state_bits(b), ref1)
    b.check_status()
    g, _ = load_golden("cfg2")
    assert_scaled_close(batch_energies(b, w.paulis, w.coeffs), g["energies"][:8], RTOL)

    eager.reset()
    eager.execute(plan2)
    ref2 = _state_bits(eager)
    gp.replay(plan2.gates1, plan2.gates2)
    _assert_same(_state_bits(b), ref2)
    e_graph = batch_energies(b, w2.paulis, w2.coeffs)
    e_eager = batch_energies(eager, w2.paulis, w2.coeffs)
    assert np.array_equal(e_graph, e_eager)
    assert len(b.update_records(0)) == len(eager.update_records(0)) > 0
    gp.replay(plan.gates1, plan.gates2)       # and back
    _assert_same(_state_bits(b), ref1)


def test_graph_replay_guards():
    from paper_1807_07914_b200 import MpsBatch, TruncationPolicy, compile_batch
    from paper_1807_07914_b200.workloads import brick_circuit

    n = 10
    progs = [brick_circuit(n, 6, np.random.default_rng(5 + s)) for s in range(3)]
    plan = compile_batch(progs, n)
    b = MpsBatch(3, n, TruncationPolicy(1e-10, 8))
    gp = b.capture(plan)
    with pytest.raises(ValueError, match="captured plan holds"):
        gp.replay(gates1=plan.gates1[:-1])
    b.ensure_capacity(2 * b.cap)               # re-allocates gamma / lam / dims
    with pytest.raises(RuntimeError, match="capture the plan again"):
        gp.replay()
    with pytest.raises(ValueError, match="empty plan"):
        b.capture(compile_batch([[]], n))

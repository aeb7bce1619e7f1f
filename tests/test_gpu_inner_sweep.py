"""The inner (Gram-space) Jacobi sweep of a block-pair visit on its own -- the batched
rotation scheme of csrc/bmps_jacobi.cuh (jac_inner: four rounds per batch, one warp per
group of 8 columns, the rest applied as 8x8 unitaries on DMMA) -- against numpy
properties that do not depend on the pair ordering: Q is unitary, G_out = Q^H G_in Q,
a sweep reduces the coupling it works on, converged / degenerate inputs are left alone.
This is the scalar core of the replacement of ``np.linalg.svd`` at mps.py:116."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

EPS = 1.1102230246251565e-16


def _sweep(G, full, tol=4 * np.sqrt(512.0) * EPS, fro=None, max_inner=1):
    import torch
    from paper_1807_07914_b200 import _native
    lib = _native.load()
    fro = float(np.sqrt(np.trace(G).real)) if fro is None else fro
    dev = torch.device("cuda:0")
    gin = torch.from_numpy(np.asfortranarray(G).T.copy()).to(dev)      # column-major 32 x 32
    gout = torch.empty_like(gin)
    q = torch.empty_like(gin)
    nrot = torch.zeros(1, dtype=torch.int32, device=dev)
    rc = lib.bmps_debug_inner_sweep(gin.data_ptr(), gout.data_ptr(), q.data_ptr(), int(full), tol,
                                    (1e-14 * fro) ** 2, fro, max_inner, nrot.data_ptr(),
                                    ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    _native.check(rc, "bmps_debug_inner_sweep")
    torch.cuda.synchronize()
    return gout.cpu().numpy().T, q.cpu().numpy().T, int(nrot.item())


def _gram(rng, grading):
    P = (rng.standard_normal((512, 32)) + 1j * rng.standard_normal((512, 32))) * grading[None, :]
    return P.conj().T @ P


def _off(G, full):
    if full:
        return np.linalg.norm(G - np.diag(np.diag(G)))
    return np.linalg.norm(G[:16, 16:])


@pytest.mark.parametrize("full", [0, 1])
@pytest.mark.parametrize("decades", [0.0, 4.0, 10.0])
def test_sweep_is_a_unitary_congruence_and_reduces_the_coupling(full, decades):
    rng = np.random.default_rng(int(10 * decades) + full)
    G = _gram(rng, 10.0 ** (-decades * np.arange(32) / 31.0))
    Gout, Q, nrot = _sweep(G, full)
    assert nrot == (496 if full else 256)
    assert np.abs(Q.conj().T @ Q - np.eye(32)).max() < 1e-14
    # entrywise against the scale of the rows / columns it mixes
    scale = np.sqrt(np.outer(np.diag(G).real, np.diag(G).real)).max()
    assert np.abs(Q.conj().T @ G @ Q - Gout).max() < 1e-13 * scale
    assert np.abs(Gout - Gout.conj().T).max() < 1e-13 * scale
    # a sweep takes the coupling it works on down; full sweeps converge quadratically
    # (a cross sweep alone is re-coupled through the two blocks' own off-diagonals)
    assert _off(Gout, full) < 0.7 * _off(G, full)
    if full:
        Gk = Gout
        for _ in range(5):
            Gk, _, _ = _sweep(Gk, full)
        assert _off(Gk, full) < 1e-6 * _off(G, full)


def test_repeated_sweeps_diagonalise_the_gram():
    rng = np.random.default_rng(5)
    G = _gram(rng, 10.0 ** (-6.0 * np.arange(32) / 31.0))
    Gout, Q, _ = _sweep(G, 1, max_inner=30)
    d = np.sqrt(np.diag(Gout).real)
    rel = np.abs(Gout - np.diag(np.diag(Gout))) / np.outer(d, d)
    fro = np.sqrt(np.trace(G).real)
    # converged in the kernel's sense: |g_ij| <= tol * min(|x_i|, |x_j|) * ||M||_F
    tol = 4 * np.sqrt(512.0) * EPS
    bound = tol * np.minimum.outer(d, d) * fro
    assert (np.abs(Gout - np.diag(np.diag(Gout))) <= 1.01 * bound + 1e-300).all()
    ev = np.sort(np.linalg.eigvalsh(G))[::-1]
    assert np.abs(np.sort(np.diag(Gout).real)[::-1] - ev).max() < 1e-12 * ev[0]
    assert rel.max() < 1.0


@pytest.mark.parametrize("full", [0, 1])
def test_converged_and_degenerate_inputs_are_left_alone(full):
    G = np.diag(10.0 ** (-np.arange(32) / 4.0)).astype(complex)
    Gout, Q, nrot = _sweep(G, full)
    assert nrot == 0 and np.array_equal(Q, np.eye(32)) and np.array_equal(Gout, G)
    # zero columns (rank-deficient panel) and columns under the noise floor never rotate
    rng = np.random.default_rng(9)
    grading = np.ones(32)
    grading[5] = 0.0
    grading[20] = 0.0
    grading[27] = 1e-16
    grading[9] = 1e-17
    G = _gram(rng, grading)
    Gout, Q, nrot = _sweep(G, full)
    assert np.isfinite(Gout).all() and np.isfinite(Q).all()
    assert np.abs(Q.conj().T @ Q - np.eye(32)).max() < 1e-14
    for dead in (5, 20):
        e = np.zeros(32)
        e[dead] = 1.0
        assert np.array_equal(Q[:, dead], e) and np.array_equal(Q[dead, :], e)

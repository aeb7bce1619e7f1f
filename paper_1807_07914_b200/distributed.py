"""Multi-GPU sharding of independent MPS work.

One process per GPU (``torchrun``), NCCL over NVLink for the single
collective the path has: the VQE energy reduction. Everything else is
embarrassingly parallel -- circuits, parameter vectors or Hamiltonian terms
are dealt round-robin to ranks (truncation makes per-item cost uneven, so
round-robin balances better than contiguous blocks) and never exchange
tensors.

Two VQE modes:
  * ``by_vector``: rank r evolves vectors r, r+G, ... and evaluates all terms
    for them; energies are scattered into a zero vector and summed with one
    allreduce (exact: each entry has exactly one non-zero contributor).
  * ``by_term``: every rank evolves the same vectors and evaluates a slice of
    the terms; per-term values are combined in term order after an
    all-gather so the left-to-right sum of ``vqe.py:89`` is preserved.
"""

from __future__ import annotations

from typing import Callable, Sequence

import numpy as np
import torch
import torch.distributed as dist


def shard(n_items: int, world: int, rank: int) -> np.ndarray:
    """Round-robin indices of the items owned by ``rank``."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    return np.arange(rank, n_items, world, dtype=np.int64)


def _device_for(group) -> torch.device:
    backend = dist.get_backend(group)
    return torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")


def allreduce_scattered(local_idx: np.ndarray, local_vals: np.ndarray, total: int, group=None) -> np.ndarray:
    """Place local values at their global indices and sum across ranks (one allreduce)."""
    buf = torch.zeros(total, dtype=torch.float64, device=_device_for(group))
    if len(local_idx):
        buf[torch.as_tensor(local_idx, device=buf.device)] = torch.as_tensor(
            np.asarray(local_vals, dtype=np.float64), device=buf.device)
    dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    return buf.cpu().numpy()


def energies_by_vector(n_vectors: int, evaluate: Callable[[np.ndarray], np.ndarray], group=None) -> np.ndarray:
    """``evaluate(indices) -> energies`` for this rank's vectors; returns all energies."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    idx = shard(n_vectors, world, rank)
    vals = evaluate(idx) if len(idx) else np.zeros(0)
    return allreduce_scattered(idx, vals, n_vectors, group)


def energies_by_term(n_vectors: int, coeffs: Sequence[float],
                     term_values: Callable[[np.ndarray], np.ndarray], group=None) -> np.ndarray:
    """``term_values(term_idx) -> [n_vectors, len(term_idx)]`` expectations for this
    rank's terms; returns sum_k c_k <P_k> per vector in term order (vqe.py:89).

    One collective for the whole batch: every rank scatters its columns into a
    zero [n_vectors, n_terms] matrix and a single allreduce(sum) assembles it
    (exact: each entry has one non-zero contributor); the weighted sums then run
    left to right on the host, as the reference's Python ``sum``."""
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    nt = len(coeffs)
    tidx = shard(nt, world, rank)
    local = term_values(tidx) if len(tidx) else np.zeros((n_vectors, 0))
    buf = torch.zeros((n_vectors, nt), dtype=torch.float64, device=_device_for(group))
    if len(tidx):
        buf[:, torch.as_tensor(tidx, device=buf.device)] = torch.as_tensor(
            np.asarray(local, dtype=np.float64).reshape(n_vectors, len(tidx)), device=buf.device)
    dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    full = buf.cpu().numpy()
    c = np.asarray([float(x) for x in coeffs], dtype=np.float64)
    if nt == 0:
        return np.zeros(n_vectors)
    # np.add.accumulate is sequential: bit-identical to the scalar left-to-right loop
    return np.add.accumulate(c[None, :] * full, axis=1)[:, -1].copy()


def vqe_energies(programs, n: int, paulis, coeffs, policy=None, group=None, mode: str = "by_vector"):
    """Distributed cfg2-style energy evaluation on this rank's GPU."""
    from .backends import simulate_batch
    from .vqe import batch_energies

    if mode == "by_vector":
        def evaluate(idx):
            batch = simulate_batch([programs[i] for i in idx], n, policy)
            return batch_energies(batch, paulis, coeffs)
        return energies_by_vector(len(programs), evaluate, group)
    if mode == "by_term":
        batch = simulate_batch(list(programs), n, policy)

        def term_values(tidx):
            sel = [paulis[t] for t in tidx]
            sidx = np.repeat(np.arange(len(programs), dtype=np.int32), len(sel))
            return batch.expectations(sidx, sel * len(programs)).reshape(len(programs), len(sel))
        return energies_by_term(len(programs), coeffs, term_values, group)
    raise ValueError(f"unknown mode {mode!r}")

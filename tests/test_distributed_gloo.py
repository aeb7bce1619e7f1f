"""World-size-2 gloo tests of the sharding / allreduce host logic (CPU only).

The per-rank compute is injected: here the CPU oracle stands in as the checker
for what each rank's GPU batch would return, so the collective composition is
verified end to end without a GPU."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1807_07914_b200.distributed import energies_by_term, energies_by_vector, shard


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, mode, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.mps_oracle import oracle_run
    from paper_1807_07914_b200.workloads import config2
    w = config2(batch=4)
    terms = w.paulis[:12]
    coeffs = w.coeffs[:12]

    def energies(idx):
        res = []
        for v in idx:
            o = oracle_run(w.programs[v], w.n, w.cutoff, w.max_bond)
            vals = o.expectations_env(terms)
            res.append(sum(c * x for c, x in zip(coeffs.tolist(), vals)))
        return np.array(res)

    if mode == "vector":
        e = energies_by_vector(4, energies)
    else:
        states = [oracle_run(p, w.n, w.cutoff, w.max_bond) for p in w.programs]
        e = energies_by_term(4, coeffs.tolist(),
                             lambda t: np.array([[s.expectations_env([terms[i] for i in t])] for s in states]).reshape(4, len(t)))
    out[rank] = e.tolist()
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["vector", "term"])
def test_world2_energies_match_single_process(mode):
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    mp.start_processes(_worker, args=(2, port, mode, out), nprocs=2, join=True, start_method="spawn")
    from oracle.mps_oracle import oracle_run
    from paper_1807_07914_b200.workloads import config2
    w = config2(batch=4)
    ref = []
    for p in w.programs:
        o = oracle_run(p, w.n, w.cutoff, w.max_bond)
        vals = o.expectations_env(w.paulis[:12])
        ref.append(sum(c * x for c, x in zip(w.coeffs[:12].tolist(), vals)))
    for r in range(2):
        np.testing.assert_allclose(out[r], ref, rtol=0, atol=1e-12)


def test_shard_round_robin():
    assert shard(10, 4, 1).tolist() == [1, 5, 9]
    allidx = np.sort(np.concatenate([shard(10, 4, r) for r in range(4)]))
    assert allidx.tolist() == list(range(10))
    with pytest.raises(ValueError):
        shard(3, 2, 2)

"""World > 1 check of the sharded paths over NCCL (run under torchrun, one GPU per
rank): cfg2 energies by vector and by term (one allreduce each) and a cfg4 shard
per rank, compared on rank 0 with the reference goldens. Used by
tests/test_gpu_multigpu.py when >= 2 GPUs are visible."""

import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main() -> None:
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    from conftest import load_golden
    from paper_1807_07914_b200 import TruncationPolicy, simulate_batch
    from paper_1807_07914_b200 import workloads as W
    from paper_1807_07914_b200.distributed import shard, vqe_energies
    w = W.config2(batch=8)
    pol = TruncationPolicy(w.cutoff, w.max_bond)
    e_vec = vqe_energies(w.programs, w.n, w.paulis, w.coeffs, pol, mode="by_vector")
    e_term = vqe_energies(w.programs, w.n, w.paulis, w.coeffs, pol, mode="by_term")
    mine = shard(64, world, rank)
    w4 = W.config4(circuits=64, indices=list(mine))
    b = simulate_batch(w4.programs, w4.n, TruncationPolicy(w4.cutoff, w4.max_bond))
    zz = b.expectations(np.arange(len(mine), dtype=np.int32), w4.paulis * len(mine))
    full = torch.zeros(64, dtype=torch.float64, device="cuda")
    full[torch.as_tensor(mine, device="cuda")] = torch.as_tensor(zz, device="cuda")
    dist.all_reduce(full)
    if rank == 0:
        g2, _ = load_golden("cfg2")
        g4, _ = load_golden("cfg4")
        ref = g2["energies"][:8]
        scale = np.max(np.abs(ref))
        out = {"world": world,
               "by_vector_err": float(np.max(np.abs(e_vec - ref)) / scale),
               "by_term_err": float(np.max(np.abs(e_term - ref)) / scale),
               "cfg4_zz_err": float(np.max(np.abs(full.cpu().numpy() - g4["zz"][:64])) / np.max(np.abs(g4["zz"][:64])))}
        print("DIST_CHECK " + json.dumps(out), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

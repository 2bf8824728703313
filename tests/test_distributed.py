"""Column-sharded bi-level projection (paper_2405_02086_b200.distributed).

CPU: world_size-2 gloo runs of the sharding logic with an oracle-backed
local backend (test-only), compared bit for bit with the single-process
oracle on the whole matrix.  GPU: the CUDA backend on simulated shards
(one device) against the single-call projection.
"""
import os
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as td
import torch.multiprocessing as tmp

from oracle import oracle as O
from paper_2405_02086_b200 import datagen, distributed
from tests.parity import check_bilevel

CASES = [("1", "inf"), ("1", "1"), ("1", "2"), ("2", "inf"), ("inf", "2")]


class OracleBackend:
    """Local steps on CPU f64 tensors through the C oracle (tests only)."""

    def norms(self, y, q):
        return torch.from_numpy(O.aggregate(y.numpy(), q).copy())

    def outer(self, v, p, eta):
        return torch.from_numpy(O.project_ball(v.numpy(), p, eta))

    def apply(self, y, x, q, v, u, flags=0):
        return torch.from_numpy(O.project_fibers(y.numpy(), q, v.numpy(), u.numpy()))

    def gather(self, v_local, group=None):
        return distributed.gather_norms(v_local, group)


def _worker(rank, world, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        y = datagen.normal(41, (23, 70), dtype=np.float64)
        split = [0, 37, 70]  # uneven column blocks
        y_local = torch.from_numpy(np.ascontiguousarray(y[:, split[rank]:split[rank + 1]]))
        for i, (p, q) in enumerate(CASES):
            eta = 0.3 * O.matrix_pq_norm(y, p, q)
            x_local, u_local, z = distributed.sharded_bilevel_project(y_local, eta, p, q, backend=OracleBackend())
            np.save(os.path.join(outdir, f"x{i}_r{rank}.npy"), x_local.numpy())
            np.save(os.path.join(outdir, f"u{i}_r{rank}.npy"), u_local.numpy())
            np.save(os.path.join(outdir, f"z{i}_r{rank}.npy"), np.array([z]))
    finally:
        td.destroy_process_group()


def test_sharded_projection_gloo_world2():
    outdir = tempfile.mkdtemp()
    port = 29500 + (os.getpid() % 1000)
    tmp.spawn(_worker, args=(2, port, outdir), nprocs=2, join=True)
    y = datagen.normal(41, (23, 70), dtype=np.float64)
    for i, (p, q) in enumerate(CASES):
        eta = 0.3 * O.matrix_pq_norm(y, p, q)
        ref = O.bilevel(y, eta, p, q)
        x = np.concatenate([np.load(os.path.join(outdir, f"x{i}_r{r}.npy")) for r in (0, 1)], axis=1)
        u = np.concatenate([np.load(os.path.join(outdir, f"u{i}_r{r}.npy")) for r in (0, 1)])
        assert np.array_equal(x.view(np.uint64), ref["X"].view(np.uint64)), (p, q)
        assert np.array_equal(u, ref["budgets"]), (p, q)
        for r in (0, 1):
            assert int(np.load(os.path.join(outdir, f"z{i}_r{r}.npy"))[0]) == ref["zero_columns"]


@pytest.mark.gpu
def test_cuda_backend_simulated_shards_match_single_call():
    import paper_2405_02086_b200 as mp
    be = distributed.CudaBackend()
    y = torch.from_numpy(datagen.uniform(42, (2000, 3000), -1.0, 1.0)).cuda()
    blocks = [(0, 1200), (1200, 3000)]
    for p, q in CASES:
        colnorm = {"1": lambda t: t.abs().double().sum(0), "2": lambda t: t.double().pow(2).sum(0).sqrt(),
                   "inf": lambda t: t.abs().double().amax(0)}[q](y)
        outer = {"1": lambda v: v.sum(), "2": lambda v: v.pow(2).sum().sqrt(), "inf": lambda v: v.amax()}[p](colnorm)
        eta = 0.2 * float(outer)
        ys = [y[:, a:b].contiguous() for a, b in blocks]
        vs = [be.norms(t, mp.norm_code(q)) for t in ys]
        v = torch.cat(vs)
        u = be.outer(v, mp.norm_code(p), eta)
        xs = [be.apply(t, torch.empty_like(t), mp.norm_code(q), vl, u[a:b]) for t, vl, (a, b) in zip(ys, vs, blocks)]
        x = torch.cat(xs, dim=1)
        x1, b1, _ = mp.bilevel_project(y, eta, p, q)
        torch.cuda.synchronize()
        if q == "inf":  # column maxima are exact: sharded == single call, bit for bit
            assert torch.equal(u, b1), (p, q)
            assert torch.equal(x.view(torch.int32), x1.view(torch.int32)), (p, q)
        else:  # l1 / l2 column sums group rows by the grid: equal to f64 rounding
            torch.testing.assert_close(u, b1, rtol=1e-12, atol=0.0)
        y_h = y.cpu().numpy()
        check_bilevel(x.cpu().numpy(), y_h, O.bilevel(y_h.astype(np.float64), eta, p, q), q)

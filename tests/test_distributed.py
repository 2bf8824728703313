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

    device = torch.device("cpu")

    def norms(self, y, q, out):
        return out.copy_(torch.from_numpy(O.aggregate(y.numpy(), q).copy()))

    def outer(self, v, p, eta, out):
        return out.copy_(torch.from_numpy(O.project_ball(v.numpy(), p, eta)))

    def apply(self, y, x, q, v, u, flags=0):
        return x.copy_(torch.from_numpy(O.project_fibers(y.numpy(), q, v.numpy(), u.numpy())))


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
        # a planned projector reused across radii, equal block widths (no gather compaction)
        y2 = datagen.uniform(43, (17, 64), -1.0, 1.0, dtype=np.float64)
        blk = torch.from_numpy(np.ascontiguousarray(y2[:, 32 * rank:32 * (rank + 1)]))
        proj = distributed.ShardedBilevelProjector(17, 32, torch.float64, "1", "inf", backend=OracleBackend())
        for k, frac in enumerate((0.05, 0.5)):
            eta = frac * O.matrix_pq_norm(y2, "1", "inf")
            out = torch.empty_like(blk)
            proj(blk, out, eta)
            np.save(os.path.join(outdir, f"p{k}_r{rank}.npy"), out.numpy())
            np.save(os.path.join(outdir, f"pz{k}_r{rank}.npy"), np.array([proj.zero_columns()]))
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
    y2 = datagen.uniform(43, (17, 64), -1.0, 1.0, dtype=np.float64)
    for k, frac in enumerate((0.05, 0.5)):
        ref = O.bilevel(y2, frac * O.matrix_pq_norm(y2, "1", "inf"), "1", "inf")
        x = np.concatenate([np.load(os.path.join(outdir, f"p{k}_r{r}.npy")) for r in (0, 1)], axis=1)
        assert np.array_equal(x.view(np.uint64), ref["X"].view(np.uint64))
        for r in (0, 1):
            assert int(np.load(os.path.join(outdir, f"pz{k}_r{r}.npy"))[0]) == ref["zero_columns"]


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
        be.plan(2000, 1800, 3000, mp._capi.MP_F32, mp.norm_code(p), mp.norm_code(q))
        vs = [be.norms(t, mp.norm_code(q), torch.empty(t.shape[1], dtype=torch.float64, device="cuda")) for t in ys]
        v = torch.cat(vs)
        u = be.outer(v, mp.norm_code(p), eta, torch.empty_like(v))
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


@pytest.mark.gpu
def test_sharded_projector_nccl_world1_graph_capture():
    """The planned projector on NCCL (world 1) inside a captured CUDA graph:
    no host sync and no C-ABI allocation per call, result equal to the
    single-call projection bit for bit (l_inf maxima are exact)."""
    import paper_2405_02086_b200 as mp
    store = td.HashStore()
    td.init_process_group("nccl", store=store, rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        y = torch.from_numpy(datagen.uniform(44, (3000, 2500), -1.0, 1.0)).cuda()
        eta = 0.1 * float(y.abs().amax(0).double().sum())
        proj = distributed.ShardedBilevelProjector(3000, 2500, torch.float32, "1", "inf")
        x = torch.empty_like(y)
        proj(y, x, eta)  # warm-up outside capture (NCCL communicator setup)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        x.zero_()
        with torch.cuda.graph(g):
            proj(y, x, eta)
        g.replay()
        torch.cuda.synchronize()
        x1, b1, z1 = mp.bilevel_project(y, eta, "1", "inf")
        assert torch.equal(x.view(torch.int32), x1.view(torch.int32))
        assert torch.equal(proj.budgets, b1)
        assert proj.zero_columns() == z1
    finally:
        td.destroy_process_group()

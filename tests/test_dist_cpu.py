"""Mode-1 sharding on the CPU.

1. The library's host-only shard layout (`tca_shard_layout`) against brute
   force: owned rows partition [0, n1), data rows are exactly the support of
   the owned columns of A_1.
2. A world-size-2 `gloo` run of the sharded CG that the GPU path executes --
   shard-local rhs from the shard's data rows, per-apply exchange of 3
   boundary mode-1 slabs with each neighbour, all-reduce of the two dot
   products -- with the arithmetic of each shard done by the CPU oracle's
   mode products on the shard's band blocks.  It must reproduce the global
   oracle CG (Fig. 2) at matched iteration count.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth

HALO = 3   # half-bandwidth of G_1 (cubic B-spline Gram), >= that of R_1 (2)


def _layout(n1, A1, r, P):
    from paper_1001_5460_b200 import tca
    return tca.shard_layout(n1, A1, r, P)


@pytest.mark.parametrize("n1,m1,P", [(12, 20, 2), (32, 64, 3), (17, 26, 4), (9, 14, 3), (128, 256, 8)])
def test_shard_layout_partition_and_data_support(n1, m1, P):
    A1 = synth.bspline_matrix(n1, m1)
    prev_hi = 0
    for r in range(P):
        lo, hi, dlo, dhi = _layout(n1, A1, r, P)
        assert lo == prev_hi and hi > lo and hi - lo >= HALO
        prev_hi = hi
        support = np.nonzero(np.any(A1[:, lo:hi] != 0.0, axis=1))[0]
        assert (dlo, dhi) == (support.min(), support.max() + 1)
        # the owned rhs rows depend on no data row outside [dlo, dhi)
        assert not np.any(A1[:dlo, lo:hi]) and not np.any(A1[dhi:, lo:hi])
    assert prev_hi == n1


def test_shard_layout_rejects_too_many_ranks():
    from paper_1001_5460_b200 import tca
    A1 = synth.bspline_matrix(8, 16)
    with pytest.raises(tca.TcaError):
        tca.shard_layout(8, A1, 0, 3)   # 8 < 3 * 3


# ------------------------------------------------------------------ gloo emulation
def _shard_apply(x_ext, blocks, G, R, lam, lo, hi, n1):
    """q_loc = (G_1[lo:hi, ext] (x) G_2 (x) ...) x_ext + lam * (R_1[lo:hi, ext] x_ext + sum_{d>0} R_d x_loc)."""
    g1, r1 = blocks
    D = len(G)
    k = oracle.mode_product(x_ext, 0, g1)
    for d in range(1, D):
        k = oracle.mode_product(k, d, G[d])
    x_loc = x_ext[HALO:HALO + hi - lo]
    reg = oracle.mode_product(x_ext, 0, r1) if R[0] is not None else np.zeros_like(k)
    for d in range(1, D):
        if R[d] is not None:
            reg = reg + oracle.mode_product(x_loc, d, R[d])
    return k + lam * reg


def _halo(x_loc, rank, P):
    """[3 ghost | own | 3 ghost] slabs from the neighbours (zero beyond the domain)."""
    shp = (HALO,) + x_loc.shape[1:]
    lo_g = torch.zeros(shp, dtype=torch.float64)
    hi_g = torch.zeros(shp, dtype=torch.float64)
    t = torch.from_numpy(np.ascontiguousarray(x_loc))
    reqs = []
    if rank > 0:
        reqs.append(dist.isend(t[:HALO].contiguous(), rank - 1))
        reqs.append(dist.irecv(lo_g, rank - 1))
    if rank + 1 < P:
        reqs.append(dist.isend(t[-HALO:].contiguous(), rank + 1))
        reqs.append(dist.irecv(hi_g, rank + 1))
    for q in reqs:
        q.wait()
    return np.concatenate([lo_g.numpy(), x_loc, hi_g.numpy()], axis=0)


def _allreduce(v):
    t = torch.tensor([v], dtype=torch.float64)
    dist.all_reduce(t)
    return float(t[0])


def _worker(rank, P, port, case, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=P)
    n, m, lam, iters = case
    A, L = synth.mode_matrices(n, m, basis="bspline", seed=1)
    n1 = n[0]
    lo, hi, dlo, dhi = _layout(n1, A[0], rank, P)
    G = [oracle.gram(a) for a in A]
    R = [oracle.gram(l) for l in L]
    # band blocks of mode 1 for the shard: rows [lo, hi) over ext columns [lo-3, hi+3)
    def block(Mfull):
        B = np.zeros((hi - lo, hi - lo + 2 * HALO))
        for i in range(lo, hi):
            for c in range(lo - HALO, hi + HALO):
                if 0 <= c < n1:
                    B[i - lo, c - lo + HALO] = Mfull[i, c]
        return B
    blocks = (block(G[0]), block(R[0]))
    # shard-local rhs from the shard's data rows only
    y = synth.data(A, n, m, seed=1)
    A_loc = [A[0][dlo:dhi, lo:hi]] + A[1:]
    b = y[dlo:dhi]
    for d, Ad in enumerate(A_loc):
        b = oracle.mode_product(b, d, np.ascontiguousarray(Ad.T))
    # Fig. 2 CG, dots all-reduced, P exchanged after every update
    x = np.zeros_like(b)
    r = b.copy()
    p = r.copy()
    rho = _allreduce(oracle.dot(r, r))
    for _ in range(iters):
        q = _shard_apply(_halo(p, rank, P), blocks, G, R, lam, lo, hi, n1)
        alpha = rho / _allreduce(oracle.dot(p, q))
        x = x + alpha * p
        r = r - alpha * q
        rho1 = _allreduce(oracle.dot(r, r))
        p = r + (rho1 / rho) * p
        rho = rho1
    np.save(os.path.join(out_dir, f"x{rank}.npy"), x)
    np.save(os.path.join(out_dir, f"b{rank}.npy"), b)
    dist.destroy_process_group()


@pytest.mark.parametrize("case,P", [(((12, 10, 9), (20, 17, 15), 1e-2, 25), 2),
                                    (((16, 6, 5, 4), (32, 12, 10, 8), 1e-3, 20), 2)])
def test_gloo_world2_sharded_cg_matches_global_oracle(case, P, tmp_path):
    port = 29500 + (os.getpid() % 1000)
    mp.start_processes(_worker, args=(P, port, case, str(tmp_path)), nprocs=P, join=True,
                       start_method="spawn")
    n, m, lam, iters = case
    A, L = synth.mode_matrices(n, m, basis="bspline", seed=1)
    o = oracle.Operator(A, L, lam)
    b_ref = o.rhs(synth.data(A, n, m, seed=1))
    b = np.concatenate([np.load(tmp_path / f"b{r}.npy") for r in range(P)], axis=0)
    assert np.linalg.norm(b - b_ref) <= 1e-13 * np.linalg.norm(b_ref)
    x_ref, k, st, _ = o.cg(b_ref, rtol=0.0, max_iters=iters)
    x = np.concatenate([np.load(tmp_path / f"x{r}.npy") for r in range(P)], axis=0)
    assert k == iters
    assert np.linalg.norm(x - x_ref) <= 1e-10 * np.linalg.norm(x_ref)

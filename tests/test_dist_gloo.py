"""Multi-rank host logic on CPU (gloo, world_size 2): the slab sharding of the last mode, the NCCL
unique-id handshake of the drop-in ``fit(..., distributed=...)``, and the exact collective pattern
the engine uses per iteration -- allreduce(sum) of the pass-A partials (M_1..M_{N-1} numerators),
allgather of the pass-B rows (M_N) and allreduce of ||Y||^2 / direct residuals -- verified against
the unsharded oracle.  (GPU multi-rank runs need >1 GPU; this round's box has one.)"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import cp_oracle as O


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sharded_mttkrps(y, factors, lo, hi):
    """What one rank's engine computes on its slab Y[..., lo:hi] (tensor_pass.cuh): pass A gives
    partial M_1..M_{N-1} (sum over the local last-mode slices), pass B gives rows lo:hi of M_N."""
    nm = len(factors)
    local = y[..., lo:hi]
    lf = list(factors[:-1]) + [factors[-1][lo:hi]]
    parts = [O.mttkrp(np.asfortranarray(local), lf, n) for n in range(1, nm)]
    rows_n = O.mttkrp(np.asfortranarray(local), lf, nm)
    return parts, rows_n


def _worker(rank, world, port, y, factors, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1205_2584_b200 import slab_bounds
        from paper_1205_2584_b200.solver import _Dist

        ctx = _Dist()
        uid = ctx.unique_id()  # rank 0 creates the NCCL id through the C ABI, all ranks receive it
        lo, hi = slab_bounds(y.shape[-1], world, rank)
        parts, rows_n = _sharded_mttkrps(y, factors, lo, hi)
        # allreduce(sum) of the packed pass-A partials, exactly one collective per pass
        pack = torch.from_numpy(np.concatenate([p.reshape(-1, order="F") for p in parts]).copy())
        dist.all_reduce(pack)
        # allgather of the (padded) pass-B row blocks
        per = -(-y.shape[-1] // world)
        pad = np.zeros((per, rows_n.shape[1]), dtype=rows_n.dtype)
        pad[: hi - lo] = rows_n
        gathered = [torch.zeros_like(torch.from_numpy(pad)) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(pad))
        mn = np.concatenate([g.numpy() for g in gathered])[: y.shape[-1]]
        # ||Y||^2 and the direct residual of the model: scalar allreduces
        ysq = torch.tensor([float(np.sum(np.abs(y[..., lo:hi]) ** 2))], dtype=torch.float64)
        dist.all_reduce(ysq)
        xr = O.reconstruct(factors)[..., lo:hi]
        rsq = torch.tensor([float(np.sum(np.abs(y[..., lo:hi] - xr) ** 2))], dtype=torch.float64)
        dist.all_reduce(rsq)
        q.put((rank, uid, lo, hi, pack.numpy(), mn, float(ysq.item()), float(rsq.item())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("dims", [(5, 4, 7), (3, 4, 2, 6), (6, 9)])
def test_two_rank_slab_collectives_match_unsharded(dims):
    rng = np.random.default_rng(len(dims))
    rank_r = 3
    factors = [rng.standard_normal((d, rank_r)) for d in dims]
    y = np.asfortranarray(O.reconstruct(factors) + 0.1 * rng.standard_normal(dims))
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, y, factors, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in range(world)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # identical NCCL id on both ranks
    assert res[0][1] == res[1][1] and len(res[0][1]) == 128
    # slabs tile the last mode
    assert res[0][2] == 0 and res[0][3] == res[1][2] and res[1][3] == dims[-1]
    full = [O.mttkrp(y, factors, n) for n in range(1, len(dims) + 1)]
    want_pack = np.concatenate([f.reshape(-1, order="F") for f in full[:-1]])
    for r in res:
        np.testing.assert_allclose(r[4], want_pack, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(r[5], full[-1], rtol=1e-12, atol=1e-12)
        assert r[6] == pytest.approx(float(np.sum(y * y)), rel=1e-13)
        assert r[7] == pytest.approx(float(np.sum((y - O.reconstruct(factors)) ** 2)), rel=1e-12)
    # both ranks hold bit-identical reduced data (identical decisions on every rank)
    np.testing.assert_array_equal(res[0][4], res[1][4])
    np.testing.assert_array_equal(res[0][5], res[1][5])


def _slab_worker(rank, world, port, path, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1205_2584_b200 import cptn, slab_bounds

        h = cptn.read_header(path)
        lo, hi = slab_bounds(h.dims[-1], world, rank)
        mine = cptn.read_slab(path, lo, hi, h)  # only this rank's byte range of the file
        per = -(-h.dims[-1] // world)
        pad = np.zeros(tuple(h.dims[:-1]) + (per,), dtype=mine.dtype, order="F")
        pad[..., : hi - lo] = mine
        flat = torch.from_numpy(np.ascontiguousarray(pad.reshape(-1, order="F")).view(np.float64))
        got = [torch.zeros_like(flat) for _ in range(world)]
        dist.all_gather(got, flat)
        if rank == 0:
            parts = [g.numpy().view(mine.dtype).reshape(pad.shape, order="F") for g in got]
            q.put(np.concatenate(parts, axis=-1)[..., : h.dims[-1]])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("complex_", [False, True])
def test_cptn_slab_byte_ranges_tile_the_file(tmp_path, complex_):
    """Each rank reads only its slab's byte range of a CPTN file (the cpf_engine_load_cptn
    arithmetic); gathered, the slabs are the tensor read_tensor returns."""
    from paper_1205_2584_b200 import cptn
    from paper_1205_2584_b200.tensor import DenseTensor

    rng = np.random.default_rng(7)
    y = rng.standard_normal((5, 4, 7))
    if complex_:
        y = y + 1j * rng.standard_normal(y.shape)
    path = tmp_path / "y.cptn"
    cptn.write_tensor(path, DenseTensor(y))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    mp.start_processes(_slab_worker, args=(2, _free_port(), str(path), q), nprocs=2, join=True, start_method="spawn")
    full = q.get(timeout=60)
    assert np.array_equal(full, cptn.read_tensor(path).data)

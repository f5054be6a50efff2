"""Host-side logic of the slab decomposition on CPU with
world_size 2 (gloo): the halo ring, the two transposes of the fused passes in
exactly the layouts the CUDA kernels use (paper_2203_02962_b200.dist.slab_layout
restates csrc/fftfused.cu TLayout), and the scalar reductions."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _exchange(chunks_send, world):
    """all-to-all of equal numpy chunks with point-to-point gloo messages."""
    rank = dist.get_rank()
    recv = [None] * world
    reqs = []
    bufs = [torch.zeros(len(chunks_send[0]) * 2, dtype=torch.float64) for _ in range(world)]
    for q in range(world):
        if q == rank:
            continue
        send = torch.from_numpy(np.ascontiguousarray(chunks_send[q]).view(np.float64).copy())
        reqs.append(dist.isend(send, q))
        reqs.append(dist.irecv(bufs[q], q))
    for r in reqs:
        r.wait()
    for q in range(world):
        recv[q] = chunks_send[q] if q == rank else bufs[q].numpy().view(np.complex128)
    return recv


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2203_02962_b200.dist import halo_planes, slab_layout, slab_range
    rng = np.random.default_rng(7)
    c, n0, n1, n2 = 2, 8, 8, 8
    glob = rng.standard_normal((c, n0, n1, n2))
    z0, nz = slab_range(n0, rank, world)
    local = glob[:, z0:z0 + nz]
    # ---- halo ring (context.cu exchange_halo): first plane -> prev, last -> next
    prev, nxt = (rank - 1) % world, (rank + 1) % world
    hlo = torch.zeros(c * n1 * n2, dtype=torch.float64)
    hhi = torch.zeros(c * n1 * n2, dtype=torch.float64)
    first = torch.from_numpy(np.ascontiguousarray(local[:, 0]).ravel())
    last = torch.from_numpy(np.ascontiguousarray(local[:, -1]).ravel())
    if world == 1:
        hhi.copy_(first)
        hlo.copy_(last)
    else:
        reqs = [dist.isend(first, prev), dist.isend(last, nxt), dist.irecv(hhi, nxt), dist.irecv(hlo, prev)]
        for r in reqs:
            r.wait()
    lo_g, hi_g = halo_planes(n0, rank, world)
    ok_halo = np.array_equal(hlo.numpy().reshape(c, n1, n2), glob[:, lo_g]) and \
        np.array_equal(hhi.numpy().reshape(c, n1, n2), glob[:, hi_g])
    # ---- transpose 1: planes -> k1 rows (pass 1 -> pass 2)
    L = slab_layout(c, n0, n1, world)
    P = L.P
    X = rng.standard_normal((c, n0, n1, P)) + 1j * rng.standard_normal((c, n0, n1, P))  # pass-1 values
    T = np.zeros(world * L.chunk_t(), dtype=np.complex128)
    for comp in range(c):
        for i0l in range(nz):
            for k1 in range(n1):
                for k2 in range(P):
                    T[L.t(k1 // L.n1l, comp, k1 % L.n1l, k2, i0l)] = X[comp, z0 + i0l, k1, k2]
    recv = _exchange([T[q * L.chunk_t():(q + 1) * L.chunk_t()] for q in range(world)], world)
    Tr = np.concatenate(recv)
    ok_t = True
    for comp in range(c):
        for k1l in range(L.n1l):
            for k2 in range(P):
                pencil = np.array([Tr[L.t(i0 // L.nzl, comp, k1l, k2, i0 % L.nzl)] for i0 in range(n0)])
                ok_t &= np.array_equal(pencil, X[comp, :, rank * L.n1l + k1l, k2])
    # ---- transpose 2: k1 rows -> planes (pass 2 -> pass 3)
    Y = rng.standard_normal((c, n0, n1, P)) + 1j * rng.standard_normal((c, n0, n1, P))
    T2 = np.zeros(world * L.chunk_t2(), dtype=np.complex128)
    for comp in range(c):
        for i0 in range(n0):
            for k1l in range(L.n1l):
                for k2 in range(P):
                    T2[L.t2(i0 // L.nzl, comp, i0 % L.nzl, k1l, k2)] = Y[comp, i0, rank * L.n1l + k1l, k2]
    recv2 = _exchange([T2[q * L.chunk_t2():(q + 1) * L.chunk_t2()] for q in range(world)], world)
    T2r = np.concatenate(recv2)
    ok_t2 = True
    for comp in range(c):
        for i0l in range(nz):
            for k1 in range(n1):
                row = np.array([T2r[L.t2(k1 // L.n1l, comp, i0l, k1 % L.n1l, k2)] for k2 in range(P)])
                ok_t2 &= np.array_equal(row, Y[comp, z0 + i0l, k1])
    # ---- peer pull (no all-to-all): every rank's send buffers readable in
    # place (all_gather stands in for the NVLink mappings); passes 2 and 3
    # address source q's chunk for this rank through the pull offsets
    def gather(buf):
        t = torch.from_numpy(buf.view(np.float64).copy())
        allb = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allb, t)
        return [b.numpy().view(np.complex128) for b in allb]
    Tall, T2all = gather(T), gather(T2)
    ok_pull = True
    for comp in range(c):
        for k1l in range(L.n1l):
            for k2 in range(P):
                pencil = []
                for i0 in range(n0):
                    q = i0 // L.nzl
                    off = L.pull_offset(rank, q, L.chunk_t())
                    pencil.append(Tall[q][off + L.t(q, comp, k1l, k2, i0 % L.nzl)])
                ok_pull &= np.array_equal(np.array(pencil), X[comp, :, rank * L.n1l + k1l, k2])
        for i0l in range(nz):
            for k1 in range(n1):
                q = k1 // L.n1l
                off = L.pull_offset(rank, q, L.chunk_t2())
                row = np.array([T2all[q][off + L.t2(q, comp, i0l, k1 % L.n1l, k2)] for k2 in range(P)])
                ok_pull &= np.array_equal(row, Y[comp, z0 + i0l, k1])
    # ---- scalar all-reduction of per-rank partial sums
    part = torch.tensor([float(np.sum(local ** 2))], dtype=torch.float64)
    dist.all_reduce(part)
    ok_red = abs(part.item() - float(np.sum(glob ** 2))) <= 1e-12 * float(np.sum(glob ** 2))
    out[rank] = (bool(ok_halo), bool(ok_t), bool(ok_t2), bool(ok_red), bool(ok_pull))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2, 4])
def test_slab_exchanges_gloo(world):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        assert out[r] == (True, True, True, True, True), (r, out[r])


def test_slab_ranges_and_halos_match_reference_wrap(oracle_mod):
    """Halo plane indices equal the reference's periodic wrap (bit-exact)."""
    from paper_2203_02962_b200.dist import halo_planes, slab_range
    n0 = 16
    og = oracle_mod.Grid((n0, 4, 4), (1.0, 1.0, 1.0), "trilinear-hex")
    nbr = og.neighbor_table()  # offsets: index 4 = (1,0,0)
    for world in (1, 2, 4, 8):
        covered = []
        for rank in range(world):
            z0, nz = slab_range(n0, rank, world)
            covered.extend(range(z0, z0 + nz))
            lo, hi = halo_planes(n0, rank, world)
            last_pixel = ((z0 + nz - 1) * 4) * 4
            assert nbr[last_pixel, 4] // 16 == hi
            prev_last = (((z0 - 1) % n0) * 4) * 4
            assert nbr[prev_last, 4] // 16 == z0 and lo == (z0 - 1) % n0
        assert covered == list(range(n0))


def _worker_2d(rank, world, port, out):
    """2-D row slabs (c5): halo rows and the half-spectrum column-chunk
    transposes of the slab spectra (csrc/context.cu d == 2, slabfft.cu with a
    unit last axis), restated with dist.slab_layout_2d: row r2c on the owner,
    padded column chunks exchanged, axis-0 transform on the column owner ==
    numpy rfft2 of the global field on those columns; and back."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2203_02962_b200.dist import halo_planes, slab_layout_2d, slab_range
    rng = np.random.default_rng(11)
    c, n0, n1 = 1, 12, 10
    glob = rng.standard_normal((c, n0, n1))
    z0, nz = slab_range(n0, rank, world)
    local = glob[:, z0:z0 + nz]
    # halo rows
    prev, nxt = (rank - 1) % world, (rank + 1) % world
    hlo = torch.zeros(c * n1, dtype=torch.float64)
    hhi = torch.zeros(c * n1, dtype=torch.float64)
    first = torch.from_numpy(np.ascontiguousarray(local[:, 0]).ravel())
    last = torch.from_numpy(np.ascontiguousarray(local[:, -1]).ravel())
    if world == 1:
        hhi.copy_(first)
        hlo.copy_(last)
    else:
        reqs = [dist.isend(first, prev), dist.isend(last, nxt), dist.irecv(hhi, nxt), dist.irecv(hlo, prev)]
        for r in reqs:
            r.wait()
    lo_g, hi_g = halo_planes(n0, rank, world)
    ok_halo = np.array_equal(hlo.numpy().reshape(c, n1), glob[:, lo_g]) and \
        np.array_equal(hhi.numpy().reshape(c, n1), glob[:, hi_g])
    # forward: row r2c into padded S, pack per destination, exchange
    L = slab_layout_2d(c, n0, n1, world)
    S = np.zeros(c * nz * world * L.nhl, dtype=np.complex128)
    rows = np.fft.rfft(local, axis=2)  # (c, nz, nh)
    for comp in range(c):
        for i0l in range(nz):
            for k1 in range(L.nh):
                S[L.s_index(comp, i0l, k1)] = rows[comp, i0l, k1]
    chunk = c * nz * L.nhl
    send = []
    for q in range(world):
        buf = np.zeros(chunk, dtype=np.complex128)
        for comp in range(c):
            for i0l in range(nz):
                for k1l in range(L.nhl):
                    buf[(comp * nz + i0l) * L.nhl + k1l] = S[L.s_index(comp, i0l, q * L.nhl + k1l)]
        send.append(buf)
    recv = _exchange(send, world)
    W = np.zeros(c * n0 * L.nhl, dtype=np.complex128)
    for q in range(world):
        for comp in range(c):
            for i0l in range(nz):
                for k1l in range(L.nhl):
                    W[L.w_index(comp, q * nz + i0l, k1l)] = recv[q][(comp * nz + i0l) * L.nhl + k1l]
    Wf = np.fft.fft(W.reshape(c, n0, L.nhl), axis=1)
    full = np.fft.rfft2(glob, axes=(1, 2))
    ok_fwd = True
    for k1l in range(L.nhl):
        k1 = rank * L.nhl + k1l
        if L.valid(k1):
            ok_fwd &= np.allclose(Wf[:, :, k1l], full[:, :, k1], rtol=0, atol=1e-12)
        else:
            ok_fwd &= np.array_equal(Wf[:, :, k1l], np.zeros((c, n0)))  # padding stays zero
    # inverse: axis-0 inverse on the columns, exchange back, row c2r
    Wi = np.fft.ifft(Wf, axis=1).reshape(-1)
    send = []
    for q in range(world):
        buf = np.zeros(chunk, dtype=np.complex128)
        for comp in range(c):
            for i0l in range(nz):
                for k1l in range(L.nhl):
                    buf[(comp * nz + i0l) * L.nhl + k1l] = Wi[L.w_index(comp, q * nz + i0l, k1l)]
        send.append(buf)
    recv = _exchange(send, world)
    S2 = np.zeros((c, nz, world * L.nhl), dtype=np.complex128)
    for q in range(world):
        for comp in range(c):
            for i0l in range(nz):
                S2[comp, i0l, q * L.nhl:(q + 1) * L.nhl] = recv[q][(comp * nz) * L.nhl + i0l * L.nhl:
                                                                    (comp * nz) * L.nhl + (i0l + 1) * L.nhl]
    back = np.fft.irfft(S2[:, :, :L.nh], n=n1, axis=2)
    ok_inv = np.allclose(back, local, rtol=0, atol=1e-12)
    out[rank] = (bool(ok_halo), bool(ok_fwd), bool(ok_inv))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2, 4])
def test_slab_2d_exchanges_gloo(world):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_2d, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        assert out[r] == (True, True, True), (r, out[r])

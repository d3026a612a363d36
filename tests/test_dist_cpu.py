"""CPU, world_size 2 and 3 over gloo: the sharded step's host logic.

Each rank fetches ITS schedule from the extension (etd_sharded_schedule — the
same records build_plan turns into device copies / NCCL send-recv) and runs it
on host buffers with gloo point-to-point messages, chunk by chunk as the device
overlaps them.  Checks: the forward exchange of every z-stage chunk lands
exactly that chunk's y rows of every z plane in the chunk's z-stage block, and
the backward exchanges + unpack rebuild the z-slab layout.  Also the NCCL
unique-id bootstrap used by bench.py (rank 0 creates, broadcast over the
process group)."""
import ctypes as C
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


NF = 13  # int64 fields per schedule record


def _schedule(L, nx, ny, nz, ns, G, r, pitch, chunks):
    cnt = C.c_int()
    assert L.etd_sharded_schedule(nx, ny, nz, ns, G, r, pitch, chunks, None, 0, C.byref(cnt)) == 0
    out = np.zeros(cnt.value * NF, dtype=np.int64)
    assert L.etd_sharded_schedule(nx, ny, nz, ns, G, r, pitch, chunks, out.ctypes.data_as(C.c_void_p), cnt.value,
                                  C.byref(cnt)) == 0
    return out.reshape(-1, NF)


def _worker(rank, world, port, shape, ns, chunks, result_q):
    import sys
    sys.path.insert(0, ROOT)
    import paper_2601_06849_b200 as etd
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        L = etd.lib()
        L.etd_sharded_schedule.argtypes = [C.c_int] * 6 + [C.c_longlong, C.c_int, C.c_void_p, C.c_int,
                                                           C.POINTER(C.c_int)]
        nx, ny, nz = shape
        pitch = (nx + 31) // 32 * 32
        z0, z1 = etd.zslab_partition(nz, world, rank)
        j0, j1 = etd.zslab_partition(ny, world, rank)
        nzr, njr = z1 - z0, j1 - j0
        F, Fz = pitch * ny * nzr, pitch * njr * nz
        rng = np.random.default_rng(0)
        U = np.zeros((ns, nz, ny, pitch))
        U[..., :nx] = rng.standard_normal((ns, nz, ny, nx))
        bufs = {0: U[:, z0:z1].reshape(-1).copy(), 1: np.zeros(ns * F), 2: np.full(2 * ns * Fz, np.nan),
                3: np.zeros(2 * ns * Fz), 4: np.zeros(2 * ns * F), 5: np.full(2 * ns * F, np.nan)}
        sched = _schedule(L, nx, ny, nz, ns, world, rank, pitch, chunks)
        # this rank's z-stage chunks: rows [a, b) of its y range, block offset in zin / wz
        spans, base, off = [], [], 0
        for k in range(chunks):
            a, b = etd.zslab_partition(njr, chunks, k) if chunks <= njr else ((k, k + 1) if k < njr else (njr, njr))
            spans.append((a, b))
            base.append(off)
            off += 2 * ns * nz * (b - a) * pitch

        def copy2d(r):
            _, _, _, db, do, dp, sb, so, sp, w, h, _, _ = [int(x) for x in r]
            for row in range(h):
                bufs[db][do + row * dp: do + row * dp + w] = bufs[sb][so + row * sp: so + row * sp + w]

        def exchange(phase, k):
            sends = [r for r in sched if r[1] == phase and r[0] == 1 and r[12] == k]
            recvs = [r for r in sched if r[1] == phase and r[0] == 2 and r[12] == k]
            reqs, landing = [], []
            tag_s, tag_r = {}, {}
            for r in sends:
                peer, b, off, cnt = int(r[2]), int(r[6]), int(r[7]), int(r[11])
                t = tag_s.get(peer, 0)
                tag_s[peer] = t + 1
                payload = torch.from_numpy(bufs[b][off:off + cnt].copy())
                if peer == rank:
                    landing.append(("self", t, payload))
                else:
                    reqs.append(dist.isend(payload, dst=peer, tag=t))
            for r in recvs:
                peer, b, off, cnt = int(r[2]), int(r[3]), int(r[4]), int(r[11])
                t = tag_r.get(peer, 0)
                tag_r[peer] = t + 1
                if peer == rank:
                    src = [x for x in landing if x[1] == t][0][2]
                    assert src.numel() == cnt, "self piece size mismatch"
                    bufs[b][off:off + cnt] = src.numpy()
                else:
                    tgt = torch.empty(cnt, dtype=torch.float64)
                    reqs.append(dist.irecv(tgt, src=peer, tag=t))
                    landing.append((b, off, tgt))
            for q in reqs:
                q.wait()
            for x in landing:
                if x[0] != "self":
                    bufs[x[0]][x[1]:x[1] + x[2].numel()] = x[2].numpy()

        for r in sched:
            if r[1] == 0:
                copy2d(r)
        for k in range(chunks):  # all forward exchanges first, as the comm stream issues them
            exchange(1, k)
        ok_fwd = True
        for k, (a, b) in enumerate(spans):
            nk = b - a
            if nk == 0:
                continue
            blk = bufs[2][base[k]: base[k] + ns * nz * nk * pitch].reshape(ns, nz, nk, pitch)
            ok_fwd &= np.array_equal(blk, U[:, :, j0 + a:j0 + b, :])
            # stand-in z-stage output of the chunk: a known function of global coordinates
            c_, z_, j_, x_ = np.meshgrid(np.arange(2 * ns), np.arange(nz), np.arange(j0 + a, j0 + b),
                                         np.arange(pitch), indexing="ij")
            bufs[3][base[k]: base[k] + 2 * ns * nz * nk * pitch] = (c_ * 1e6 + z_ * 1e4 + j_ * 1e2 + x_).reshape(-1)
            exchange(2, k)
        for k in range(chunks):
            if spans[k][1] == spans[k][0]:
                exchange(2, k)  # an empty chunk of this rank still receives its peers' rows
        for r in sched:
            if r[1] == 3:
                copy2d(r)
        w = bufs[5].reshape(2 * ns, nzr, ny, pitch)
        c_, z_, j_, x_ = np.meshgrid(np.arange(2 * ns), np.arange(z0, z1), np.arange(ny), np.arange(pitch),
                                     indexing="ij")
        ok_back = np.array_equal(w, c_ * 1e6 + z_ * 1e4 + j_ * 1e2 + x_)
        # the level-2 y stack pass reads the slab straight from the receive blocks
        # (etd_sharded_recv_rows): the same values as the unpacked slab
        L.etd_sharded_recv_rows.argtypes = [C.c_int] * 5 + [C.c_longlong, C.c_int, C.c_void_p]
        tab = np.zeros(3 * ny, dtype=np.int64)
        assert L.etd_sharded_recv_rows(ny, nz, ns, world, rank, pitch, chunks, tab.ctypes.data_as(C.c_void_p)) == 0
        via = np.empty_like(w)
        for c in range(2 * ns):
            for zl in range(nzr):
                for j in range(ny):
                    o = tab[3 * j] + c * tab[3 * j + 1] + zl * tab[3 * j + 2]
                    via[c, zl, j] = bufs[4][o:o + pitch]
        ok_back = ok_back and np.array_equal(via, w)
        # NCCL unique-id bootstrap (bench.py): rank 0 creates, everyone receives
        obj = [etd.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ok_id = isinstance(obj[0], bytes) and len(obj[0]) == 128
        result_q.put((rank, bool(ok_fwd), bool(ok_back), ok_id))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,shape,ns,chunks", [(2, (13, 11, 9), 2, 4), (3, (21, 7, 10), 1, 4),
                                                   (2, (33, 16, 16), 1, 1), (3, (9, 5, 6), 2, 3)])
def test_sharded_schedule_over_gloo(world, shape, ns, chunks):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, shape, ns, chunks, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_fwd, ok_back, ok_id in res:
        assert ok_fwd, f"rank {rank}: forward exchange layout"
        assert ok_back, f"rank {rank}: backward exchange + unpack layout"
        assert ok_id


def test_partition_balanced():
    import paper_2601_06849_b200 as etd
    for n, G in ((1023, 8), (1023, 3), (7, 7), (10, 4)):
        parts = [etd.zslab_partition(n, G, r) for r in range(G)]
        assert parts[0][0] == 0 and parts[-1][1] == n
        assert all(parts[i][1] == parts[i + 1][0] for i in range(G - 1))
        sizes = [b - a for a, b in parts]
        assert max(sizes) - min(sizes) <= 1
    with pytest.raises(etd.ConfigError):
        etd.zslab_partition(4, 5, 0)

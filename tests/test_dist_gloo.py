"""Multi-process host logic of the N > 1 path on CPU (gloo, world size 2 and 3).

The NCCL path moves the same opaque byte tensors: the exported query ciphertext is
broadcast from rank 0 and the per-rank score ciphertexts are gathered to rank 0.
Here the bytes are the oracle's own ciphertext residues, so a bit flip anywhere in
the plumbing fails the comparison."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2604_00546_b200 import dist as hdd


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, payload, results):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A = 7
        a0, a1 = hdd.shard_range(A, rank, world)
        # query broadcast: only rank 0 holds the bytes
        src = torch.from_numpy(payload.copy()) if rank == 0 else None
        got = hdd.broadcast_bytes(src, payload.nbytes, "cpu")
        ok_bcast = bool((got.numpy() == payload).all())
        # each rank "produces" one score ciphertext per local aggregate: tagged copies
        local = torch.from_numpy(np.concatenate([np.roll(payload, a) for a in range(a0, a1)]) if a1 > a0
                                 else np.zeros(0, np.uint8))
        per = payload.nbytes
        gathered = hdd.gather_bytes(local, ((A + world - 1) // world) * per, 0)
        mx = hdd.max_over_ranks(float(rank + 1), "cpu")
        if rank == 0:
            flat = torch.cat(gathered).numpy()
            want = np.concatenate([np.roll(payload, a) for a in range(A)])
            results.put(("gather", bool((flat == want).all())))
        results.put(("bcast", ok_bcast))
        results.put(("range", (a0, a1)))
        results.put(("max", mx))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_broadcast_gather_and_sharding(world, oracle_mod):
    o = oracle_mod.Oracle(6, 3)
    s, s_ntt = o.secret_key()
    z = np.linspace(-1, 1, o.ns)
    ct = o.encrypt(s_ntt, o.encode(z, 2.0 ** 45, 3), 1000)
    payload = ct.view(np.uint8).ravel()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, payload, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = [q.get() for _ in range(3 * world + 1)]
    assert all(v for k, v in res if k in ("gather", "bcast"))
    ranges = sorted(v for k, v in res if k == "range")
    assert ranges[0][0] == 0 and ranges[-1][1] == 7
    assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
    assert all(v == world for k, v in res if k == "max")


def _split_worker(rank, world, port, r_all, results):
    """bench.py --split-baby on gloo: each rank fills its slice of the baby steps (here taken
    from the oracle's r) into its chunk; all_gather_into_tensor must reassemble r in order."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n1, ct = r_all.shape[0], r_all[0].size
        chunk, i0, i1 = hdd.baby_slice(n1, rank, world)
        mine = torch.zeros(chunk * ct, dtype=torch.int64)
        if i1 > i0:
            mine[: (i1 - i0) * ct] = torch.from_numpy(r_all[i0:i1].reshape(-1).view(np.int64))
        full = torch.empty(world * chunk * ct, dtype=torch.int64)
        dist.all_gather_into_tensor(full, mine)
        if rank == 0:
            got = full.numpy()[: n1 * ct].view(np.uint64).reshape(r_all.shape)
            results.put(("split", bool((got == r_all).all())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_split_baby_all_gather(world, oracle_mod):
    o = oracle_mod.Oracle(6, 3)
    s, s_ntt = o.secret_key()
    n1 = 8
    steps, keys = o.keyset(s_ntt, list(range(1, n1)))
    qct = o.encrypt(s_ntt, o.encode(np.linspace(-1, 1, o.ns), 2.0 ** 45, 3), 1000)
    r_all = o.baby_steps(qct, n1, steps, keys)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_split_worker, args=(r, world, port, r_all, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert q.get() == ("split", True)
    assert [hdd.baby_slice(n1, r, world)[1:] for r in range(world)][0][0] == 0


def _membership_worker(rank, world, port, cts, mods, results):
    """bench.py --scenario membership at N > 1: each rank sums (EvalAddMany) its comparison
    ciphertexts, the partial sums are gathered to rank 0, which runs the membership tail."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a0, a1 = hdd.shard_range(cts.shape[0], rank, world)
        part = np.zeros(cts.shape[1:], dtype=object)
        for a in range(a0, a1):
            part = (part + cts[a].astype(object)) % mods
        local = torch.from_numpy(part.astype(np.uint64).view(np.uint8).ravel().copy())
        got = hdd.gather_bytes(local, local.numel(), 0)
        if rank == 0:
            results.put(("parts", [g.numpy().view(np.uint64).reshape(cts.shape[1:]) for g in got]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_membership_partial_sums(world, oracle_mod):
    o = oracle_mod.Oracle(6, 3)
    s, s_ntt = o.secret_key()
    rng = np.random.default_rng(world)
    cts = np.stack([o.encrypt(s_ntt, o.encode(rng.uniform(0, 1, o.ns) * 1e-3, 2.0 ** 45, 2), 50 + a)
                    for a in range(5)])
    mods = np.array(o.p.moduli[:2], dtype=object)[None, :, None]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_membership_worker, args=(r, world, port, cts, mods, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    _, parts = q.get()
    st, keys = o.keyset(s_ntt, [1 << k for k in range(o.log_n - 1)])
    assert (o.membership(np.stack(parts), st, keys) == o.membership(cts, st, keys)).all()


def _exchange_worker(rank, world, port, qbytes, cts, results):
    """bench.py's per-step exchange (StepExchange) on gloo with oracle ciphertext payloads: the
    C-ABI export is replaced by a byte copy into the send slab at the pointer StepExchange hands
    out; every step reuses the same buffers (no allocation) and sizes never travel."""
    import ctypes

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A = cts.shape[0]
        a0, a1 = hdd.shard_range(A, rank, world)
        ob = cts[0].nbytes
        xch = hdd.StepExchange(qbytes.nbytes, hdd.shard_sizes(A, world), ob, "cpu")
        ptrs = (xch.qbuf.data_ptr(), xch.send.data_ptr(),
                [b.data_ptr() for b in xch.recv] if xch.recv is not None else None)

        def export_into(a, ptr, cap):  # stands in for hd_ciphertext_export_level(.., device dst)
            src = np.ascontiguousarray(cts[a]).view(np.uint8)
            assert cap == src.nbytes
            ctypes.memmove(ptr, src.ctypes.data, cap)

        ok = True
        for step in range(3):
            if rank == 0:
                xch.qbuf.copy_(torch.from_numpy(np.roll(qbytes, step)))
            got_q = xch.broadcast_query().numpy()
            ok = ok and bool((got_q == np.roll(qbytes, step)).all())
            views = xch.gather(list(range(a0, a1)), export_into)
            same = (xch.qbuf.data_ptr(), xch.send.data_ptr(),
                    [b.data_ptr() for b in xch.recv] if xch.recv is not None else None) == ptrs
            ok = ok and same
            if rank == 0:
                flat = [v for per in views for v in per]
                assert len(flat) == A
                for a, (p_, n_) in enumerate(flat):
                    buf = (ctypes.c_uint8 * n_).from_address(p_)
                    ok = ok and bool((np.frombuffer(buf, np.uint8) == cts[a].view(np.uint8).ravel()).all())
        results.put(("exchange", rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_step_exchange_fixed_buffers(world, oracle_mod):
    """The N > 1 timed step's collectives (a1 query broadcast, a9 gather of 1-limb result
    exports) on persistent buffers sized from the static shard map, with ragged shards
    (A = 7 over 2 or 3 ranks): every gathered ciphertext arrives bit for bit in aggregate order."""
    o = oracle_mod.Oracle(6, 3)
    s, s_ntt = o.secret_key()
    rng = np.random.default_rng(world)
    cts = np.stack([np.ascontiguousarray(o.encrypt(s_ntt, o.encode(rng.uniform(-1, 1, o.ns), 2.0 ** 45, 3),
                                                   300 + a)[:, :1]) for a in range(7)])  # 1-limb exports
    qct = o.encrypt(s_ntt, o.encode(np.linspace(-1, 1, o.ns), 2.0 ** 45, 3), 1000)
    qbytes = qct.view(np.uint8).ravel().copy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, qbytes, cts, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = [q.get() for _ in range(world)]
    assert all(ok for _, _, ok in res), res

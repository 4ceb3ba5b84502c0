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

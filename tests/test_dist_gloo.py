"""World-size-2 gloo tests of the multi-rank host logic (CPU): sharding covers every packet
exactly once, and update deltas planned on rank 0 and broadcast leave every rank's tables
byte-identical to a ctx that applied the same ops locally."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import tang_inputs as ti


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2601_03187_b200 import dist as D, tang as T, train as TR
        R = ti.classbench_ruleset("acl", 3000, 9)
        sigs = TR.tuple_signatures(R)
        blob = T.pack_blob(sigs, ti.random_weights(7, 64, 1, len(sigs), 0))
        ctx = T.Ctx(R, blob, device=-1)
        ref = T.Ctx(R, blob, device=-1)                  # applies the ops locally
        new = ti.classbench_ruleset("fw", 400, 10)
        new["id"] += 50000
        rng = np.random.default_rng(3)
        for win in range(4):
            dels = rng.choice(R["id"][win * 500:(win + 1) * 500], 100, replace=False)
            ops = T.make_ops(new[win * 100:(win + 1) * 100], deletes=dels)
            st, nb = D.broadcast_update(ctx, ops)
            ref.update_plan(ops)
            assert nb > 0
            if rank == 0:
                assert (st[:100] == 0).all()
            assert ctx.stats()["checksum"] == ref.stats()["checksum"]
            assert D.checksums_agree(ctx)
            dg = D.window_digests(ctx)                   # the bench's per-window replica check
            assert dg.numel() == world and bool((dg == dg[0]).all())
            assert int(dg[rank]) & ((1 << 64) - 1) == ref.mirror_digest()
        # a replica that diverged is caught by the digest check
        div = T.Ctx(R, blob, device=-1)
        if rank == 1:
            div.update_plan(T.make_ops(deletes=[int(R["id"][2999])]))
        dg = D.window_digests(div)
        assert int(dg[0]) != int(dg[1])
        # NUMA binding degrades to None without NVML / GPUs (CPU box)
        assert D.bind_numa_local(0) is None or isinstance(D.bind_numa_local(0), list)
        # shards cover [0, n) exactly once
        for n in (0, 1, 7, 1000003):
            a, b = D.shard(n, rank, world)
            got = [None] * world
            dist.all_gather_object(got, (a, b))
            cover = sorted(got)
            assert cover[0][0] == 0 and cover[-1][1] == n
            assert all(cover[i][1] == cover[i + 1][0] for i in range(world - 1))
        assert D.max_over_ranks(float(rank)) == world - 1
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, traceback.format_exc()))


def test_delta_broadcast_and_sharding_world2():
    ctxmp = mp.get_context("spawn")
    q = ctxmp.Queue()
    port = _free_port()
    ps = [ctxmp.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=240) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res

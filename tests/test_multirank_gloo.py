"""Multi-rank host logic on CPU (world_size 2 and 3, gloo, 127.0.0.1).

What the N > 1 GPU path does per rank, exercised without GPUs:
  * the partition plan from the C-ABI (`nbody_plan`, host-only) gives each rank a
    contiguous slice; the slices tile [0, n) with padding only at the tail;
  * rank 0's NCCL unique id (host-only `nbody_nccl_unique_id`) reaches every rank
    through the torch process group (broadcast_object_list), as in bench.py;
  * the in-place all-gather of equal `slot`-sized packet slices reassembles the
    global j array in global particle order (emulated with gloo all_gather);
  * per-rank forces on the own i-range (oracle) concatenate to the full evaluation;
  * block time steps: per-rank minima of t_i + dt_i (and the level-count rule the
    library uses for them) reduced with MIN give the global t_next, and the ranks'
    active sets partition the global active set;
  * bench.py's timing reduction is a MAX over ranks.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        from paper_2509_19294_b200 import binding, inputs
        oracle.set_threads(1)
        m, x, v = inputs.parity_round(*inputs.plummer(n, 77))
        p = binding.plan(n, world, rank)
        i0, i1, slot = p["i0"], p["i1"], p["slot"]
        # 1) NCCL id broadcast through the process group
        obj = [binding.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ids = [None] * world
        dist.all_gather_object(ids, obj[0])
        assert len(obj[0]) == 128 and all(i == ids[0] for i in ids)
        # 2) packet exchange: each rank fills its slot-sized slice (own particles,
        #    zero-mass padding after n), an all-gather of equal slices in rank order
        pk = np.zeros((slot, 8), dtype=np.float32)
        pk[:, 0:3] = 1e18
        k = i1 - i0
        pk[:k, 0:3] = x[:, i0:i1].T
        pk[:k, 3] = m[i0:i1]
        pk[:k, 4:7] = v[:, i0:i1].T
        parts = [torch.empty((slot, 8), dtype=torch.float32) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(pk))
        full = torch.cat(parts).numpy()
        assert np.array_equal(full[:n, 0:3], x.T.astype(np.float32))
        assert np.array_equal(full[:n, 3], m.astype(np.float32))
        assert np.all(full[n:, 3] == 0)
        # 3) per-rank forces on the own i-range concatenate to the full result
        a, j = oracle.forces(m, x, v, 1e-6, idx=np.arange(i0, i1))
        got = [None] * world
        dist.all_gather_object(got, (i0, i1, a, j))
        if rank == 0:
            got.sort(key=lambda t: t[0])
            a_all = np.concatenate([g[2] for g in got], axis=1)
            j_all = np.concatenate([g[3] for g in got], axis=1)
            af, jf = oracle.forces(m, x, v, 1e-6)
            assert np.array_equal(a_all, af) and np.array_equal(j_all, jf)
        # 4) block time steps (R#28): every rank's minimum of t_i + dt_i over its own range,
        #    reduced with MIN across ranks (the ncclAllReduce of block_run), is the global
        #    t_next, and the ranks' active sets partition the global one
        lev, _ = oracle.block_init_levels(*oracle.forces(m, x, v, 1e-6), 1 / 64, 20, 0.01)
        due = (1 << (20 - lev.astype(np.int64)))          # t_i = 0: next time of particle i
        tmin = torch.tensor([int(due[i0:i1].min()) if i1 > i0 else 2**62], dtype=torch.int64)
        dist.all_reduce(tmin, op=dist.ReduceOp.MIN)
        assert int(tmin) == int(due.min())
        mine = [int(i) for i in np.nonzero(due[i0:i1] == int(tmin))[0] + i0]
        act = [None] * world
        dist.all_gather_object(act, mine)
        assert sorted(sum(act, [])) == [int(i) for i in np.nonzero(due == due.min())[0]]
        #    later block times: the library derives each rank's t_next from its level counts
        #    (next multiple of the finest occupied level's step after the block time t,
        #    every particle last active at the last multiple of its own step); MIN over
        #    ranks of that equals the global min of t_i + dt_i
        rng = np.random.default_rng(5)
        lev2 = rng.integers(0, 8, size=n).astype(np.int64)
        for t in (0, 3 * (1 << 17), (1 << 20) - (1 << 13), 5 * (1 << 12)):
            d = 1 << (20 - lev2)
            due2 = (t // d) * d + d
            cnt = np.bincount(lev2[i0:i1], minlength=21)
            occ = np.nonzero(cnt)[0]
            if occ.size:
                dmin = 1 << (20 - int(occ.max()))
                local = (t // dmin + 1) * dmin
            else:
                local = 2**62
            assert occ.size == 0 or local == int(due2[i0:i1].min())
            tn = torch.tensor([local], dtype=torch.int64)
            dist.all_reduce(tn, op=dist.ReduceOp.MIN)
            assert int(tn) == int(due2.min()), (t, int(tn), int(due2.min()))
        # 5) max-over-ranks timing reduction (bench.py)
        t = torch.tensor([10.0 + rank, 1.0 * rank], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        assert t.tolist() == [10.0 + world - 1, float(world - 1)]
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # noqa: BLE001
        q.put((rank, f"FAIL {type(e).__name__}: {e}"))


@pytest.mark.parametrize("world,n", [(2, 1000), (3, 2049), (2, 512)])
def test_multirank_host_logic(world, n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(r[1] == "ok" for r in res), res

"""Multi-process (gloo, world_size 2, CPU) checks of the sharding host logic used by bench.py:
units are disjoint and cover the global batch, inputs regenerated per unit are bit-identical to
the unsharded generation, the timing reduction is a max over ranks, the strong split's uneven
gather is trimmed per rank, and `bench.py --gpus 2` starts its own two ranks."""
import json
import os
import subprocess
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2411_10958_b200 import shard, synth


def _free_port():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    B, Hq, Hkv, N, d = 2, 4, 2, 64, 64
    units = shard.rank_units(rank, world, B, Hkv)
    qs, ks, vs = synth.make_qkv(B, Hq, Hkv, N, d, kind="structured", seed=3, units=units)
    t = shard.max_over_ranks(1.0 + rank, world)
    gathered = [None] * world
    dist.all_gather_object(gathered, units)
    # validation gather of the per-rank outputs (here: a stand-in [B, Hq, N, d] tensor per rank)
    out = qs.view(B, Hq, N, d).float() + rank
    parts = shard.gather_outputs(out, world)
    def recompute(r):    # rank r's first unit, regenerated from its seed (what bench.py's rank 0 does)
        u0 = shard.rank_units(r, world, B, Hkv)[0]
        return synth.make_qkv(B, Hq, Hkv, N, d, kind="structured", seed=3, units=[u0])[0][0].float() + r
    bad = shard.first_unit_check(parts, recompute)
    dist.destroy_process_group()
    q.put((rank, units, t, gathered, qs.sum().item(), ks[0].numpy().copy(), vs[-1].numpy().copy(), bad))


def test_two_rank_sharding():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in procs], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    all_units = res[0][3][0] + res[0][3][1]
    assert len(set(all_units)) == len(all_units) == 2 * 2 * 2          # disjoint, complete
    assert sorted(all_units) == [(b, h) for b in range(4) for h in range(2)]
    assert res[0][2] == res[1][2] == 2.0                                # max over ranks
    assert res[0][7] == [] and res[1][7] == []                          # gathered parts in rank order
    # a rank's units regenerate exactly the slice of the unsharded (global batch 4) tensors
    qf, kf, vf = synth.make_qkv(4, 4, 2, 64, 64, kind="structured", seed=3)
    assert (res[1][5] == kf[2, 0].numpy()).all()     # rank 1, first unit = (b=2, h=0)
    assert (res[0][6] == vf[1, 1].numpy()).all()     # rank 0, last unit = (b=1, h=1)


def test_split_units_balanced():
    units = [(b, h) for b in range(3) for h in range(5)]
    parts = [shard.split_units(units, r, 4) for r in range(4)]
    assert sum(parts, []) == units
    assert max(map(len, parts)) - min(map(len, parts)) <= 1
    with pytest.raises(ValueError):
        shard.rank_units(2, 2, 1, 1)


def _strong_worker(rank, world, port, q):
    """Strong split of a fixed unit list (north-star C5 shape, scaled down) with an odd unit count:
    each rank builds its share as [n_units, grp, N, d], a stand-in output per unit (the test's own
    arithmetic, not the product), the padded gather and rank 0's first-unit check."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    B, Hq, Hkv, N, d = 3, 4, 1, 32, 64                   # 3 units: ranks own 1 and 2
    grp = Hq // Hkv
    units = shard.split_units(shard.all_units(B, Hkv), rank, world)
    qs, ks, vs = synth.make_qkv(B, Hq, Hkv, N, d, kind="iid", seed=5, units=units)
    out = (qs.float() * ks.float()[:, None]).reshape(len(units), grp, N, d)
    parts = shard.gather_units(out, len(units), world)
    bad = None
    if rank == 0:
        def recompute(r):
            u0 = shard.split_units(shard.all_units(B, Hkv), r, world)[0]
            qu, ku, _ = synth.make_qkv(B, Hq, Hkv, N, d, kind="iid", seed=5, units=[u0])
            return (qu.float() * ku.float()[:, None])[0]
        bad = shard.first_unit_check(parts, recompute)
    tot = shard.sum_over_ranks(len(units), world)
    dist.destroy_process_group()
    q.put((rank, units, [tuple(p.shape) for p in parts], bad, tot))


def test_two_rank_strong_split_and_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_strong_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=120) for _ in procs], key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0][1] + res[1][1] == [(0, 0), (1, 0), (2, 0)]
    assert res[0][2] == [(1, 4, 32, 64), (2, 4, 32, 64)]          # trimmed to each rank's count
    assert res[0][3] == []                                        # bitwise first-unit check passes
    assert res[0][4] == res[1][4] == 3.0


def test_bench_starts_its_own_ranks():
    """`python bench.py --gpus 2` outside torchrun re-executes itself under torch.distributed.run
    (127.0.0.1), one process per GPU; --dist-check stops right after the process group is up.  On a
    CPU box the group is gloo; the default multi-GPU workload is the strong split of C5."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--dist-check"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = sorted((json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")), key=lambda x: x["rank"])
    assert [x["rank"] for x in lines] == [0, 1]
    assert all(x["world"] == 2 and x["config"] == "c5_b8" and x["scaling"] == "strong" and x["reduce_ok"]
               for x in lines)
    assert [x["n_units"] for x in lines] == [128, 128]            # C5: 8 x 32 units split evenly
    assert lines[0]["first_unit"] == [0, 0] and lines[1]["first_unit"] == [4, 0]

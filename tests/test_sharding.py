"""Block sharding: assignment, rank-local structure, and the shard exchange.

CPU tests run the host logic and a world_size-2 gloo all-gather of packed shards; the GPU test checks that
two ranks' shards combined equal the unsharded step bit-for-bit (every per-block reduction is fixed-order).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_02016_b200.shampoo import build_layout
from paper_2602_02016_b200.sharded import assign_units, local_groups, packed_positions, units_of
from tests.golden.cases import MINI, RAGGED, llama_953m


@pytest.mark.parametrize("world", [1, 2, 3, 8])
@pytest.mark.parametrize("shapes,b", [(MINI, 16), (RAGGED, 8), (llama_953m(), 1024)])
def test_assignment_covers_each_block_once(shapes, b, world):
    layers, specs = build_layout(shapes, b)
    units = units_of(layers)
    a = assign_units(units, world)
    flat = sorted(i for r in a for i in r)
    assert flat == list(range(len(units)))
    assert a == assign_units(units, world)  # deterministic
    loads = [sum(units[i].cost for i in r) for r in a]
    # LPT bound: max load <= mean + largest single cost
    assert max(loads) <= sum(loads) / world + max(u.cost for u in units)


def test_953m_balance_8_ranks():
    layers, _ = build_layout(llama_953m(), 1024)
    units = units_of(layers)
    loads = [sum(units[i].cost for i in r) for r in assign_units(units, 8)]
    assert max(loads) / (sum(loads) / 8) < 1.02


@pytest.mark.parametrize("world", [2, 4])
def test_local_groups_partition_global_groups(world):
    layers, specs = build_layout(RAGGED, 8)
    units = units_of(layers)
    a = assign_units(units, world)
    seen = {}
    for r in range(world):
        owned = {(units[i].layer_id, units[i].idx) for i in a[r]}
        lspecs, slot_of, gids = local_groups(specs, owned)
        for lg, (sp, gi) in enumerate(zip(lspecs, gids)):
            assert (sp.dim, sp.exponent) == (specs[gi].dim, specs[gi].exponent)
            # local order = global order restricted
            pos = [specs[gi].members.index(m) for m in sp.members]
            assert pos == sorted(pos)
            for slot, m in enumerate(sp.members):
                assert slot_of[m].group == lg and slot_of[m].slot == slot
                assert m not in seen
                seen[m] = r
    assert set(seen) == {m for sp in specs for m in sp.members}


def _flat_index(layers, offsets, unit):
    lay = layers[unit.layer_id]
    base = offsets[unit.layer_id]
    if lay.is_matrix:
        (r0, r1), (c0, c1) = lay.layout.block_spans[unit.idx]
        n = lay.shape[1]
        return np.array([base + r * n + c for r in range(r0, r1) for c in range(c0, c1)])
    s, e = lay.chunk_bounds[unit.idx]
    return np.arange(base + s, base + e)


def _worker(rank, world, port, shapes, b, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    layers, _ = build_layout(shapes, b)
    units = units_of(layers)
    a = assign_units(units, world)
    sizes = [int(np.prod(s)) for s in shapes]
    offsets = np.concatenate([[0], np.cumsum(sizes)])
    total = int(offsets[-1])
    # "updated" flat params: only owned blocks are valid on this rank (value = global flat index + 1)
    theta = np.full(total, -1.0)
    truth = np.arange(total, dtype=np.float64) + 1.0
    order = [i for i in a[rank] if units[i].matrix] + [i for i in a[rank] if not units[i].matrix]
    for i in order:
        ix = _flat_index(layers, offsets, units[i])
        theta[ix] = truth[ix]
    maxp = max(int(packed_positions(units, r)[-1]) for r in a)
    pos = packed_positions(units, a[rank])
    send = np.zeros(maxp)
    for k, i in enumerate(order):  # pack (the CUDA pack kernel's layout)
        send[pos[k]:pos[k + 1]] = theta[_flat_index(layers, offsets, units[i])]
    recv = [torch.zeros(maxp, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(recv, torch.from_numpy(send))
    for r in range(world):  # unpack every rank's shard
        ordr = [i for i in a[r] if units[i].matrix] + [i for i in a[r] if not units[i].matrix]
        pr = packed_positions(units, a[r])
        buf = recv[r].numpy()
        for k, i in enumerate(ordr):
            theta[_flat_index(layers, offsets, units[i])] = buf[pr[k]:pr[k + 1]]
    q.put((rank, bool(np.array_equal(theta, truth))))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("shapes,b", [(MINI, 16), (RAGGED, 8)])
def test_gloo_world2_shard_exchange(shapes, b):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, shapes, b, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: True, 1: True}


@pytest.mark.gpu
def test_two_shards_equal_unsharded_step_bitwise():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2602_02016_b200.shampoo import ShampooConfig, SolverConfig, init_state, step
    from paper_2602_02016_b200.sharded import ShardedDash

    rng = np.random.default_rng(0)
    shapes = [(96, 64), (64,), (40, 72), (130, 33)]
    params = [torch.tensor(rng.standard_normal(s), dtype=torch.float32, device="cuda") for s in shapes]
    grads = [torch.tensor(rng.standard_normal(s), dtype=torch.float32, device="cuda") for s in shapes]
    cfg = ShampooConfig(block_size=32, solver=SolverConfig(tolerance=0.0, max_iters=10))
    st = init_state(params, cfg)
    ref, _ = step(st, [p.clone() for p in params], grads, cfg, seed=5)
    ref_flat = torch.cat([r.reshape(-1) for r in ref])
    shards = [ShardedDash(params, cfg, rank=r, world=2) for r in range(2)]
    outs = [sh.step_local([p.clone() for p in params], grads, seed=5).clone() for sh in shards]
    merged = torch.cat([p.reshape(-1) for p in params]).clone()
    layers, _ = build_layout(shapes, 32)
    units = units_of(layers)
    sizes = [int(np.prod(s)) for s in shapes]
    offsets = np.concatenate([[0], np.cumsum(sizes)])
    for r, sh in enumerate(shards):
        for i in sh.assignment[r]:
            ix = torch.tensor(_flat_index(layers, offsets, units[i]), device="cuda")
            merged[ix] = outs[r][ix]
    assert torch.equal(merged, ref_flat)


def _world2_cfg(nx):
    """nx = 3 also carries graft momentum (owner-only packed momentum next to the packed Adam state)."""
    from paper_2602_02016_b200.shampoo import GraftConfig, ShampooConfig, SolverConfig

    return ShampooConfig(block_size=32, solver=SolverConfig(tolerance=0.0, max_iters=10),
                         graft=GraftConfig(beta1=0.9 if nx == 3 else 0.0))


def _sharded_worker(rank, world, port, q, nx=2):
    """One rank of a world-2 ShardedDash: the full step (accumulate, refresh, apply, C-ABI pack, all-gather,
    unpack) on cuda:0 over gloo (host-staged exchange), three steps, then the flat parameters go back."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2602_02016_b200.shampoo import ShampooConfig, SolverConfig
    from paper_2602_02016_b200.sharded import ShardedDash

    rng = np.random.default_rng(0)
    shapes = [(96, 64), (64,), (40, 72), (130, 33)]
    params = [torch.tensor(rng.standard_normal(s), dtype=torch.float32, device="cuda") for s in shapes]
    grads = [[torch.tensor(rng.standard_normal(s), dtype=torch.float32, device="cuda") for s in shapes]
             for _ in range(3)]
    cfg = _world2_cfg(nx)
    opt = ShardedDash(params, cfg, rank=rank, world=world, exchange_chunks=nx)
    total = sum(int(np.prod(s)) for s in shapes)
    assert opt.state.runtime.adam.numel() < total  # owner-only Adam state
    events = {}
    for gs in grads:
        opt.step(params, gs, seed=5, events=events)
    torch.cuda.synchronize()
    q.put((rank, torch.cat([p.reshape(-1) for p in params]).cpu().numpy(), len(events.get("exchanged", []))))
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("nx", [1, 2, 3])
def test_sharded_step_world2_equals_single_gpu_bitwise(nx):
    """ShardedDash.step end to end on 2 ranks == the 1-GPU step, bit for bit, on both ranks:
    one all-gather after the step (nx = 1) or nx exchange chunks overlapped with the next chunk's solves."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2602_02016_b200.shampoo import ShampooConfig, SolverConfig, init_state, step

    rng = np.random.default_rng(0)
    shapes = [(96, 64), (64,), (40, 72), (130, 33)]
    params = [torch.tensor(rng.standard_normal(s), dtype=torch.float32, device="cuda") for s in shapes]
    grads = [[torch.tensor(rng.standard_normal(s), dtype=torch.float32, device="cuda") for s in shapes]
             for _ in range(3)]
    cfg = _world2_cfg(nx)
    st = init_state(params, cfg)
    cur = [p.clone() for p in params]
    for gs in grads:
        cur, st = step(st, cur, gs, cfg, seed=5)
    want = torch.cat([c.reshape(-1) for c in cur]).cpu().numpy()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_sharded_worker, args=(r, 2, port, q, nx)) for r in range(2)]
    for p in procs:
        p.start()
    res = {r: (flat, nex) for r, flat, nex in (q.get(timeout=300) for _ in procs)}
    for p in procs:
        p.join(timeout=60)
    for r in range(2):
        assert res[r][1] == 3
        np.testing.assert_array_equal(res[r][0], want)


def _failing_worker(rank, world, port, q):
    """Rank 1 raises inside its refresh (a tolerance its precision cannot reach); rank 0 must not hang."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    from paper_2602_02016_b200.linalg import PrecisionMode
    from paper_2602_02016_b200.shampoo import ShampooConfig, SolverConfig
    from paper_2602_02016_b200.sharded import ShardedDash

    rng = np.random.default_rng(1)
    shapes = [(64, 64), (64, 64)]
    params = [torch.tensor(rng.standard_normal(s), dtype=torch.float32, device="cuda") for s in shapes]
    grads = [torch.tensor(rng.standard_normal(s), dtype=torch.float32, device="cuda") for s in shapes]
    tol = 1e-12 if rank == 1 else 0.0
    cfg = ShampooConfig(block_size=32, solver=SolverConfig(method="cn", tolerance=tol, max_iters=4,
                                                           precision=PrecisionMode.EMULATED32))
    opt = ShardedDash(params, cfg, rank=rank, world=world)
    try:
        opt.step(params, grads)
        q.put((rank, "ok"))
    except Exception as exc:  # noqa: BLE001
        q.put((rank, type(exc).__name__))
    dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_step_error_reaches_every_rank():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_failing_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "RuntimeError", 1: "ConvergenceError"}

"""World-size-2 (and 4) CPU test of the sharded path's host logic over torch.distributed/gloo.

Each process is one rank: it owns the contiguous slice of the state selected by the
most-significant qubit digits, asks the library's shard planner (sv_shard_plan) what to do
for every gate, applies local gates to its slice with the oracle (on the local register),
and for sharded targets exchanges its slice with the partner (gloo send/recv) and combines
psi <- U[b][b] psi + U[b][1-b] psi_partner on the local indices whose local controls match
(SURVEY.md §8(e) rule iii; the combine arithmetic is restated here, independently of the
CUDA combine kernel).  The gathered result must equal O-2 on the full register."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import blocksim as O2
from sv_inputs import Gate, random_circuit, random_state, hadamard, shift_x, haar_unitary


def _local_digits(n_local, dims, D_local):
    i = np.arange(D_local)
    out = []
    for q in range(n_local):
        out.append((i // int(np.prod(dims[:q], dtype=np.int64))) % dims[q])
    return out


def _worker(rank, world, port, dims, gates, psi0, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2410_17876_b200 as P
    s = int(np.log2(world))
    n = len(dims)
    nl = n - s
    L = int(np.prod(dims[:nl]))
    psi = psi0[rank * L:(rank + 1) * L].copy()
    dg = _local_digits(nl, dims, L)
    exchanges = 0
    for g in gates:
        action, partner, beta = P.shard_plan(dims, world, rank, g.target, g.ctrl, g.vals)
        if action == 1:
            continue
        lc = [(c, v) for c, v in zip(g.ctrl, g.vals) if c < nl]
        if action == 0:
            O2.apply(psi, dims[:nl], Gate(g.target, tuple(c for c, _ in lc), tuple(v for _, v in lc), g.U))
            continue
        other = np.empty_like(psi)
        mine = torch.from_numpy(psi.view(np.float64).copy())
        theirs = torch.from_numpy(other.view(np.float64))
        reqs = [dist.isend(mine, partner), dist.irecv(theirs, partner)]
        for r in reqs:
            r.wait()
        other = theirs.numpy().view(np.complex128)
        ok = np.ones(L, dtype=bool)
        for c, v in lc:
            ok &= dg[c] == v
        a, b = g.U[beta, beta], g.U[beta, 1 - beta]
        psi = np.where(ok, a * psi + b * other, psi)
        exchanges += 1
    out = [torch.zeros(2 * L, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(out, torch.from_numpy(psi.view(np.float64).copy()))
    # the NCCL bootstrap path of bench.py: rank 0's 128-byte id reaches every rank
    idt = torch.arange(128, dtype=torch.uint8) if rank == 0 else torch.zeros(128, dtype=torch.uint8)
    dist.broadcast(idt, 0)
    if rank == 0:
        q.put((np.concatenate([t.numpy().view(np.complex128) for t in out]), exchanges,
               bool(torch.equal(idt, torch.arange(128, dtype=torch.uint8)))))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_host_logic_gloo(world):
    dims = [3, 2, 4, 2, 2, 2]
    D = int(np.prod(dims))
    _, gates = random_circuit(4242 + world, dims, 80, max_ctrl=2)
    rng = np.random.default_rng(world)
    gates += [Gate(5, (), (), hadamard()), Gate(4, (0,), (2,), haar_unitary(2, rng)),
              Gate(1, (5, 4), (1, 0), shift_x(2, 1)), Gate(5, (3,), (1,), shift_x(2, 1))]
    psi0 = random_state(D, 11)
    ref = O2.run(dims, gates, psi0)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000) + world
    procs = [ctx.Process(target=_worker, args=(r, world, port, dims, gates, psi0, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, exchanges, id_ok = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert exchanges > 0 and id_ok
    assert np.max(np.abs(got - ref)) < 1e-12


def _replay_worker(rank, world, port, dims, gates, psi0, swap, block, q):
    """Replay the library's own sharded schedule (sv_shard_schedule: rules ii-vi — predicates,
    local phases, rank relabelling, qubit remapping, exchanges — then the readback's layout
    restore) on this rank's numpy slice: local gate lists through O-2 on the local register, qubit
    swaps and exchanges as gloo send/recv with the partner the schedule names."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2410_17876_b200 as P
    s = int(np.log2(world))
    n = len(dims)
    nl = n - s
    ldims = dims[:nl]
    L = int(np.prod(ldims))
    b = np.cumprod([1] + ldims[:-1])
    dg = _local_digits(nl, dims, L)
    ops, lrank = P.sv.shard_schedule(dims, world, rank, gates, block=block, swap=swap)
    psi = psi0[rank * L:(rank + 1) * L].copy()      # initial layout: rank r holds logical slice r

    def sendrecv(arr, partner):
        mine = torch.from_numpy(arr.view(np.float64).copy())
        theirs = torch.zeros_like(mine)
        reqs = [dist.isend(mine, partner), dist.irecv(theirs, partner)]
        for r in reqs:
            r.wait()
        return theirs.numpy().view(np.complex128)

    kinds = {"local": 0, "swap": 0, "exchange": 0}
    for op in ops:
        kinds[op["kind"]] += 1
        if op["kind"] == "local":
            O2.run_inplace(psi, ldims, [Gate(t, c, v, U) for t, c, v, U in op["gates"]])
        elif op["kind"] == "swap":
            # rule vi: trade the half whose local digit k differs from this rank's sharded digit j
            # (runs of b_k amplitudes at m 2 b_k + (1 - beta) b_k) for the partner's matching half
            k, beta = op["k"], op["beta"]
            idx = np.arange(L)
            give = ((idx // b[k]) % 2) == 1 - beta
            psi[give] = sendrecv(psi[give].copy(), op["partner"])
        else:
            t, c, v, U = op["gates"][0]
            beta = op["beta"]
            other = sendrecv(psi, op["partner"])
            ok = np.ones(L, dtype=bool)
            for cc, vv in zip(c, v):
                if cc < nl:
                    ok &= dg[cc] == vv
            psi = np.where(ok, U[beta, beta] * psi + U[beta, 1 - beta] * other, psi)
    out = [torch.zeros(2 * L, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(out, torch.from_numpy(psi.view(np.float64).copy()))
    if rank == 0:
        full = np.empty(L * world, dtype=np.complex128)
        for r, t in enumerate(out):                  # physical rank r holds logical slice lrank[r]
            full[lrank[r] * L:(lrank[r] + 1) * L] = t.numpy().view(np.complex128)
        q.put((full, kinds))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("swap", [True, False])
def test_sharded_schedule_replayed_over_gloo(world, swap):
    """Rules iv-vi through the library's planner on CPU ranks: the schedule
    each rank gets from sv_shard_schedule, replayed over gloo, equals O-2 on the full register."""
    dims = [3, 2, 4, 2, 2, 2]
    D = int(np.prod(dims))
    _, gates = random_circuit(5151 + world, dims, 80, max_ctrl=2)
    rng = np.random.default_rng(world + 7)
    y = np.array([[0, -1j], [1j, 0]])
    gates += [Gate(5, (), (), hadamard()), Gate(4, (0,), (2,), haar_unitary(2, rng)),
              Gate(5, (), (), shift_x(2, 1)), Gate(4, (5,), (1,), y),                  # relabels
              Gate(5, (), (), np.diag([1, np.exp(0.7j)])), Gate(4, (1,), (1,), np.diag([np.exp(0.2j), 1])),
              Gate(1, (5, 4), (1, 0), shift_x(2, 1)), Gate(5, (3,), (1,), shift_x(2, 1))]
    psi0 = random_state(D, 12)
    ref = O2.run(dims, gates, psi0)
    ctx = mp.get_context("spawn")
    for block in (True, False):
        q = ctx.Queue()
        port = 29700 + (os.getpid() % 500) + 10 * world + (2 if swap else 0) + (1 if block else 0)
        procs = [ctx.Process(target=_replay_worker, args=(r, world, port, dims, gates, psi0, swap, block, q))
                 for r in range(world)]
        for p in procs:
            p.start()
        got, kinds = q.get(timeout=180)
        for p in procs:
            p.join(timeout=60)
            assert p.exitcode == 0
        assert np.max(np.abs(got - ref)) < 1e-12, (block, kinds)
        assert kinds["swap" if swap else "exchange"] > 0

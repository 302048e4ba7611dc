"""The sharded (multi-GPU) path's host logic on CPU.

libqvg plans a sharded circuit as a list of steps (qvg_shard_schedule): local
ops with rank predicates, pairwise half-shard exchanges, local qubit swaps.
Here the same steps are executed on CPU shards — local ops through the oracle
(test infrastructure), exchanges as numpy copies in one process, and over
torch.distributed `gloo` with world_size 2 and 4 in separate processes — and
the gathered state must equal the unsharded oracle bit for bit (the
reference's worker-count invariance, reference tests/acceptance.cpp:196-242)."""
import os
import socket

import numpy as np
import pytest

from conftest import gate_array
from oracle.oracle import GATE_DTYPE

STEP_DTYPE = np.dtype([("type", "<u4"), ("rank_mask", "<u4"), ("rank_value", "<u4"), ("gpos", "<u4"),
                       ("lpos", "<u4"), ("lpos2", "<u4"), ("op", GATE_DTYPE)])
assert STEP_DTYPE.itemsize == 104


XCHUNK_DTYPE = np.dtype([("round", "<u4"), ("partner", "<u4"), ("offset", "<u8"), ("bytes", "<u8")])
assert XCHUNK_DTYPE.itemsize == 24


def exchange_plan(n, world, rank, step, chunk_bytes, precision=128):
    """libqvg's copy-transport chunk plan for one exchange step on one rank
    (qvg_exchange_plan, the plan the NCCL and virtual-shard transports run)."""
    import ctypes

    import paper_2508_15545_b200 as qv

    lib = ctypes.CDLL(qv.LIBQVG)
    st = np.ascontiguousarray(np.asarray(step).reshape(1), STEP_DTYPE)
    cnt = ctypes.c_uint64(0)
    vp = ctypes.c_void_p
    args = [ctypes.c_uint32(n), ctypes.c_uint32(world), ctypes.c_uint32(rank), ctypes.c_uint32(precision),
            vp(st.ctypes.data), ctypes.c_uint64(chunk_bytes)]
    rc = lib.qvg_exchange_plan(*args, None, ctypes.c_uint64(0), ctypes.byref(cnt))
    if rc:
        lib.qvg_last_error.restype = ctypes.c_char_p
        raise ValueError(lib.qvg_last_error().decode())
    out = np.zeros(cnt.value, XCHUNK_DTYPE)
    rc = lib.qvg_exchange_plan(*args, vp(out.ctypes.data), ctypes.c_uint64(out.size), ctypes.byref(cnt))
    assert rc == 0
    return out


def plan_exchange(n, world, shards, st, chunk_bytes):
    """Execute one exchange step on in-process shards through libqvg's chunk
    plans: chunk i of rank r and chunk i of its partner trade places (what the
    NCCL transport's grouped send/recv does, and the virtual-shard copies)."""
    raw = [s.view(np.uint8) for s in shards]
    plans = [exchange_plan(n, world, r, st, chunk_bytes) for r in range(world)]
    for r in range(world):
        for i, c in enumerate(plans[r]):
            p = int(c["partner"])
            if p < r:
                continue
            d = plans[p][i]
            assert int(d["partner"]) == r and d["bytes"] == c["bytes"] and d["round"] == c["round"]
            a = slice(int(c["offset"]), int(c["offset"] + c["bytes"]))
            b = slice(int(d["offset"]), int(d["offset"] + d["bytes"]))
            tmp = raw[r][a].copy()
            raw[r][a] = raw[p][b]
            raw[p][b] = tmp


def schedule(qv, circuit, world, canonicalize=True, batch=1):
    raw = qv.shard_schedule(circuit.n_qubits, world, circuit.gates(), canonicalize, batch)
    return np.frombuffer(raw.tobytes(), STEP_DTYPE)


# --- batched exchange (QVG_STEP_MULTI_EXCHANGE) helpers ---------------------------------
def pext(r, mask):
    out, i = 0, 0
    for b in range(32):
        if (mask >> b) & 1:
            out |= ((r >> b) & 1) << i
            i += 1
    return out


def pdep(v, mask):
    out, i = 0, 0
    for b in range(32):
        if (mask >> b) & 1:
            out |= ((v >> i) & 1) << b
            i += 1
    return out


def multi_geometry(st):
    """(rank-bit mask, local positions in the mask's bit order)."""
    k = int(st["lpos2"])
    return int(st["gpos"]), [(int(st["lpos"]) >> (8 * i)) & 0xFF for i in range(k)]


def region(L, pos, v):
    """Local indices whose bits at pos (in order) read v, ascending."""
    x = np.arange(1 << L, dtype=np.int64)
    val = np.zeros_like(x)
    for i, p in enumerate(pos):
        val |= ((x >> p) & 1) << i
    return x[val == v]


def half_indices(L, lpos):
    """Local indices with bit lpos = 0, ascending (one side of an exchange)."""
    p = np.arange(1 << (L - 1), dtype=np.int64)
    low = (1 << lpos) - 1
    return ((p & ~low) << 1) | (p & low)


def swap_local_bits(shard, a, b):
    L = int(np.log2(shard.size))
    idx = np.arange(shard.size)
    ba, bb = (idx >> a) & 1, (idx >> b) & 1
    src = idx ^ ((ba ^ bb) << a) ^ ((ba ^ bb) << b)
    return shard[src]


def run_local_steps(oracle, L, shard, rank, steps):
    for st in steps:
        if st["type"] == 0 and (rank & st["rank_mask"]) == st["rank_value"]:
            oracle.apply(L, shard, st["op"].reshape(1))
        elif st["type"] == 2:
            shard[:] = swap_local_bits(shard, int(st["lpos"]), int(st["lpos2"]))


def emulate(oracle, n, world, steps, chunk_bytes=None):
    """All shards in one process; exchange = swap of half-shards (or, with
    chunk_bytes, libqvg's copy-transport chunk plan)."""
    g = int(np.log2(world))
    L = n - g
    shards = [np.zeros(1 << L, np.complex128) for _ in range(world)]
    shards[0][0] = 1.0
    half = 1 << (L - 1)
    for st in steps:
        if chunk_bytes is not None and st["type"] in (1, 3):
            plan_exchange(n, world, shards, st, chunk_bytes)
        elif st["type"] == 1:
            bit = 1 << (int(st["gpos"]) - L)
            lpos = int(st["lpos"])
            base = half_indices(L, lpos)
            for r in range(world):
                if r & bit:
                    continue
                p = r | bit  # r sends its local-bit-lpos=1 half, p its bit=0 half
                ri, pi = base | (1 << lpos), base
                mine, theirs = shards[r][ri].copy(), shards[p][pi].copy()
                shards[r][ri], shards[p][pi] = theirs, mine
        elif st["type"] == 3:
            # amplitude (r, x): its local bits at pos become r's swapped rank
            # bits and vice versa
            mask, pos = multi_geometry(st)
            k = len(pos)
            new = [a.copy() for a in shards]
            for r in range(world):
                w = pext(r, mask)
                for v in range(1 << k):
                    src = region(L, pos, v)
                    dst_rank = (r & ~mask) | pdep(v, mask)
                    dst = region(L, pos, w)
                    new[dst_rank][dst] = shards[r][src]
            shards = new
        else:
            for r in range(world):
                run_local_steps(oracle, L, shards[r], r, [st])
    return np.concatenate(shards)


CIRCUITS = [
    ("u3_ladder_circuit", (10, 4, 3)),
    ("random_circuit", (9, 200, 9)),
    ("haar_sweep_circuit", (12, 2)),
    ("grid_circuit", (3, 4, 6, 1)),
    ("qft_circuit", (10, 4)),
]


def build(qv, fn, args):
    out = getattr(qv, fn)(*args)
    return out[0] if isinstance(out, tuple) else out


@pytest.mark.parametrize("batch", [1, 4])
@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("fn,args", CIRCUITS)
def test_schedule_emulated_bit_identical(qv, oracle, world, fn, args, batch):
    c = build(qv, fn, args)
    steps = schedule(qv, c, world, batch=batch)
    if batch == 1 or world == 2:
        assert 3 not in set(steps["type"])
    want = oracle.simulate(c.n_qubits, gate_array(c))
    got = emulate(oracle, c.n_qubits, world, steps)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("chunk", [16, 48, 1 << 20])
@pytest.mark.parametrize("batch", [1, 4])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_copy_transport_plan_emulated_bit_identical(qv, oracle, world, batch, chunk):
    """Every exchange executed through libqvg's chunk plan (qvg_exchange_plan,
    the NCCL copy transport's send/recv list), with chunks that split runs
    (16 / 48 B) or hold whole runs, reproduces the oracle bit for bit."""
    for fn, args in [("u3_ladder_circuit", (10, 3, 5)), ("random_circuit", (9, 150, 2))]:
        c = build(qv, fn, args)
        steps = schedule(qv, c, world, batch=batch)
        assert (steps["type"] == 1).any() or (steps["type"] == 3).any()
        got = emulate(oracle, c.n_qubits, world, steps, chunk_bytes=chunk)
        assert np.array_equal(got, oracle.simulate(c.n_qubits, gate_array(c))), (fn, world, batch, chunk)


def test_copy_transport_plan_geometry(qv):
    """The plan of one exchange: a pairwise step sends exactly the amplitudes
    whose local bit lpos differs from the rank's gpos bit (2^(L-1) amplitudes,
    runs of 2^lpos, split at chunk_bytes); a k-qubit batched step sends
    (1 - 2^-k) of the shard in 2^k - 1 rounds, round t with rank ^ pdep(t)."""
    n, world = 12, 4
    L = 10
    st = np.zeros(1, STEP_DTYPE)[0]
    st["type"], st["gpos"], st["lpos"] = 1, 11, 7
    for rank in range(world):
        for chunk in (16, 1000 * 16, 1 << 20):
            plan = exchange_plan(n, world, rank, st, chunk)
            assert set(plan["partner"]) == {rank ^ 2} and set(plan["round"]) == {1}
            assert plan["bytes"].max() <= chunk and plan["bytes"].sum() == (1 << (L - 1)) * 16
            amps = np.concatenate([np.arange(o, o + b, 16) // 16 for o, b in zip(plan["offset"], plan["bytes"])])
            sendbit = 0 if rank & 2 else 1
            assert np.array_equal(amps, half_indices(L, 7) | (sendbit << 7))
    mt = np.zeros(1, STEP_DTYPE)[0]
    mt["type"], mt["gpos"], mt["lpos"], mt["lpos2"] = 3, 0b11, 9 | (8 << 8), 2
    for rank in range(world):
        plan = exchange_plan(n, world, rank, mt, 1 << 20)
        assert list(np.unique(plan["round"])) == [1, 2, 3]
        for t in (1, 2, 3):
            part = plan[plan["round"] == t]
            assert set(part["partner"]) == {rank ^ pdep(t, 0b11)}
            amps = np.concatenate([np.arange(o, o + b, 16) // 16 for o, b in zip(part["offset"], part["bytes"])])
            assert np.array_equal(amps, region(L, [9, 8], pext(rank, 0b11) ^ t))
        assert plan["bytes"].sum() == (1 - 2 ** -2) * (1 << L) * 16
    with pytest.raises(ValueError):
        exchange_plan(n, world, 0, st, 8)            # chunk not a multiple of 16
    bad = st.copy()
    bad["gpos"] = 3                                  # a local qubit is not an exchange
    with pytest.raises(ValueError):
        exchange_plan(n, world, 0, bad, 1 << 20)


def test_batched_exchange_moves_fewer_bytes(qv):
    """Config 4's circuit at 4 and 8 shards: batched exchanges (1 - 2^-k of a
    shard each) move less data than pairwise ones (1/2 each)."""
    for n, world in [(34, 4), (35, 8)]:
        c = qv.u3_ladder_circuit(n, 20, 1)
        moved = {}
        for batch in (1, 4):
            s = schedule(qv, c, world, canonicalize=False, batch=batch)
            vol = 0.0
            for st in s:
                if st["type"] == 1:
                    vol += 0.5
                elif st["type"] == 3:
                    vol += 1 - 2.0 ** -int(st["lpos2"])
            moved[batch] = vol
            if batch == 4:
                multi = s[s["type"] == 3]
                assert len(multi) > 0
                L = n - int(np.log2(world))
                for st in multi:
                    mask, pos = multi_geometry(st)
                    assert bin(mask).count("1") == len(pos) >= 2
                    assert min(pos) >= max(L - 12, L // 2) and len(set(pos)) == len(pos)
        assert moved[4] < 0.85 * moved[1], (n, world, moved)


def test_schedule_shape(qv):
    # local-only circuit: no exchange; a global target: one exchange; a global
    # control: a rank-predicated local op; a diagonal global gate: no exchange.
    n = 6
    sch = lambda text: schedule(qv, qv.parse_circuit(f"qubits {n}\n{text}\n"), 2, canonicalize=False)
    s = sch("h 0\ncx 1 2")
    assert list(s["type"]) == [0, 0]
    s = sch("h 5")
    assert list(s["type"]) == [1, 0] and s[0]["gpos"] == 5 and s[0]["lpos"] == 4
    s = sch("cx 5 0")
    assert list(s["type"]) == [0] and s[0]["rank_mask"] == 1 and s[0]["rank_value"] == 1
    s = sch("cz 0 5\nrz 5 0.3\nt 5")
    assert 1 not in list(s["type"])
    full = schedule(qv, qv.parse_circuit(f"qubits {n}\nh 5\n"), 2, canonicalize=True)
    assert list(full["type"]).count(1) == 2  # the exchange and its undo


def test_victim_choice_cuts_exchanges(qv):
    """Config 4 at full width: the Belady victim choice among the high local
    qubits needs far fewer half-shard exchanges than always swapping with
    L-1 (79 / 119 / 159 for 20 layers at 2 / 4 / 8 shards)."""
    for n, world, limit in [(33, 2, 45), (34, 4, 90), (35, 8, 135)]:
        s = schedule(qv, qv.u3_ladder_circuit(n, 20, 1), world, canonicalize=False)
        ex = s[s["type"] == 1]
        L = n - int(np.log2(world))
        assert len(ex) <= limit, (n, world, len(ex))
        assert ex["lpos"].min() >= max(L - 12, L // 2)  # blocks of >= 2^20 amplitudes


# --- multi-process: gloo, world_size 2 and 4 -----------------------------------------------
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _plan_worker(rank, world, port, fn, args, q, batch, chunk):
    """One rank of the NCCL copy transport over gloo: every exchange step runs
    libqvg's chunk plan for this rank (qvg_exchange_plan) — per chunk a
    grouped isend of the chunk and irecv into a scratch buffer, then the
    scratch copied into place, exactly the qvg_shard.hpp copy_exchange
    sequence with NCCL replaced by gloo."""
    import sys

    import torch
    import torch.distributed as dist

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import paper_2508_15545_b200 as qv
    from oracle.oracle import Oracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        oracle = Oracle()
        c = build(qv, fn, args)
        n = c.n_qubits
        L = n - int(np.log2(world))
        steps = schedule(qv, c, world, batch=batch)
        shard = np.zeros(1 << L, np.complex128)
        if rank == 0:
            shard[0] = 1.0
        raw = shard.view(np.uint8)
        chunks = 0
        for st in steps:
            if st["type"] in (1, 3):
                for ch in exchange_plan(n, world, rank, st, chunk):
                    a, b = int(ch["offset"]), int(ch["offset"] + ch["bytes"])
                    send = torch.from_numpy(raw[a:b].copy())
                    scratch = torch.empty_like(send)
                    reqs = [dist.isend(send, int(ch["partner"])), dist.irecv(scratch, int(ch["partner"]))]
                    for r in reqs:
                        r.wait()
                    raw[a:b] = scratch.numpy()
                    chunks += 1
            else:
                run_local_steps(oracle, L, shard, rank, [st])
        parts = [torch.empty(2 << L, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(shard.view(np.float64).copy()))
        if rank == 0:
            got = np.concatenate([p.numpy().view(np.complex128) for p in parts])
            want = oracle.simulate(n, gate_array(c))
            q.put((bool(np.array_equal(got, want)), chunks))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,batch,chunk", [(2, 1, 48), (4, 1, 1 << 20), (4, 4, 64)])
def test_gloo_copy_transport_plan_bit_identical(world, batch, chunk):
    """The copy transport's libqvg chunk plan executed by real processes over
    gloo (world 2 / 4, pairwise and batched exchanges) equals the oracle."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    for fn, args in [("u3_ladder_circuit", (10, 3, 5)), ("random_circuit", (8, 120, 4))]:
        port = _free_port()
        procs = [ctx.Process(target=_plan_worker, args=(r, world, port, fn, args, q, batch, chunk))
                 for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(180)
            assert p.exitcode == 0
        ok, chunks = q.get(timeout=10)
        assert ok and chunks > 0, (fn, world, batch, chunk)


def _worker(rank, world, port, fn, args, q, batch=1):
    import sys

    import torch
    import torch.distributed as dist

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import paper_2508_15545_b200 as qv
    from oracle.oracle import Oracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        oracle = Oracle()
        c = build(qv, fn, args)
        n = c.n_qubits
        L = n - int(np.log2(world))
        steps = schedule(qv, c, world, batch=batch)
        shard = np.zeros(1 << L, np.complex128)
        if rank == 0:
            shard[0] = 1.0
        half = 1 << (L - 1)
        for st in steps:
            if st["type"] == 1:  # pairwise half-shard exchange with the partner rank
                bit = 1 << (int(st["gpos"]) - L)
                lpos = int(st["lpos"])
                partner = rank ^ bit
                sendbit = 0 if (rank & bit) else 1
                idx = half_indices(L, lpos) | (sendbit << lpos)
                send = torch.from_numpy(shard[idx].view(np.float64).copy())
                recv = torch.empty_like(send)
                reqs = [dist.isend(send, partner), dist.irecv(recv, partner)]
                for r in reqs:
                    r.wait()
                shard[idx] = recv.numpy().view(np.complex128)
            elif st["type"] == 3:  # batched: 2^k - 1 XOR rounds of region swaps
                mask, pos = multi_geometry(st)
                w = pext(rank, mask)
                for t in range(1, 1 << len(pos)):
                    partner = rank ^ pdep(t, mask)
                    idx = region(L, pos, w ^ t)
                    send = torch.from_numpy(shard[idx].view(np.float64).copy())
                    recv = torch.empty_like(send)
                    reqs = [dist.isend(send, partner), dist.irecv(recv, partner)]
                    for r in reqs:
                        r.wait()
                    shard[idx] = recv.numpy().view(np.complex128)
            else:
                run_local_steps(oracle, L, shard, rank, [st])
        parts = [torch.empty(2 << L, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(shard.view(np.float64).copy()))
        if rank == 0:
            got = np.concatenate([p.numpy().view(np.complex128) for p in parts])
            want = oracle.simulate(n, gate_array(c))
            q.put(bool(np.array_equal(got, want)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,batch", [(2, 1), (4, 1), (4, 4)])
def test_gloo_multiprocess_bit_identical(world, batch):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    for fn, args in [("u3_ladder_circuit", (10, 3, 5)), ("random_circuit", (8, 120, 4))]:
        port = _free_port()
        procs = [ctx.Process(target=_worker, args=(r, world, port, fn, args, q, batch)) for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(120)
            assert p.exitcode == 0
        assert q.get(timeout=10) is True


# --- peer-memory transport protocol (k_xchg over CUDA IPC) on CPU ----------------------
# Each rank's shard is a shared-memory tensor mapped into every process (the
# CUDA IPC mapping of qvg_shard.hpp's open_peers). An exchange is the k_xchg
# protocol: barrier, each rank of the pair updates its own half of the x0
# range in BOTH shards (fused with the gate that triggered the exchange when
# the next step targets the swapped-in qubit), barrier. Ownership is disjoint,
# so the real concurrent processes here must reproduce the oracle bit for bit.
def _pair_gate(oracle, op, lo, hi):
    """The reference pair formula on vectors (lo[i], hi[i]) via the oracle:
    pack them as the two halves of a 2m-amplitude state, target its top qubit."""
    m = lo.size
    k = int(np.log2(m))
    z = np.concatenate([lo, hi])
    g = np.zeros(1, GATE_DTYPE)
    g["kind"], g["target"], g["control"], g["u"] = 0, k, -1, op["u"]
    oracle.apply(k + 1, z, g)
    return z[:m], z[m:]


def _xchg_role(oracle, shards, L, lpos, rank_a, rank_b, role, gate):
    """One rank's share of k_xchg (qvg_kernels.cuh K7)."""
    x0 = half_indices(L, lpos)
    quarter = x0.size // 2
    x0 = x0[role * quarter:(role + 1) * quarter]
    x1 = x0 | (1 << lpos)
    a, b = shards[rank_a], shards[rank_b]
    a0, a1, b0, b1 = a[x0].copy(), a[x1].copy(), b[x0].copy(), b[x1].copy()
    if gate is None:
        a[x1], b[x0] = b0, a1
        return
    pred = lambda r: (r & int(gate["rank_mask"])) == int(gate["rank_value"])
    op = gate["op"]
    on = np.ones(x0.size, bool)
    if int(op["kind"]) == 1:
        on = ((x0 >> int(op["control"])) & 1).astype(bool)
    na0, na1, nb0, nb1 = a0, b0, a1, b1
    if pred(rank_a):
        lo, hi = _pair_gate(oracle, op, a0, b0)
        na0, na1 = np.where(on, lo, a0), np.where(on, hi, b0)
    if pred(rank_b):
        lo, hi = _pair_gate(oracle, op, a1, b1)
        nb0, nb1 = np.where(on, lo, a1), np.where(on, hi, b1)
    a[x0], a[x1], b[x0], b[x1] = na0, na1, nb0, nb1


def _mxchg_role(shards, L, mask, pos, rank):
    """One rank's share of k_mxchg (qvg_kernels.cuh K8): for every round t,
    the half of the bases this rank owns, swapped between its shard and the
    partner's."""
    k = len(pos)
    w = pext(rank, mask)
    for t in range(1, 1 << k):
        wp = w ^ t
        partner = rank ^ pdep(t, mask)
        mine, theirs = region(L, pos, wp), region(L, pos, w)  # same base order
        half = mine.size // 2
        sl = slice(0, half) if w < wp else slice(half, mine.size)
        a = shards[rank][mine[sl]].copy()
        b = shards[partner][theirs[sl]].copy()
        shards[rank][mine[sl]] = b
        shards[partner][theirs[sl]] = a


def _peer_worker(rank, world, port, fn, args, tensors, q, batch=1):
    import sys

    import torch.distributed as dist

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    sys.path.insert(0, os.path.join(root, "tests"))
    import paper_2508_15545_b200 as qv
    from oracle.oracle import Oracle

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        oracle = Oracle()
        c = build(qv, fn, args)
        n = c.n_qubits
        L = n - int(np.log2(world))
        shards = [t.numpy().view(np.complex128) for t in tensors]  # every rank's shard, mapped
        steps = schedule(qv, c, world, batch=batch)
        fused = 0
        i = 0
        while i < len(steps):
            st = steps[i]
            if st["type"] == 1:
                bit = 1 << (int(st["gpos"]) - L)
                lpos = int(st["lpos"])
                nxt = steps[i + 1] if i + 1 < len(steps) else None
                gate = None
                if (nxt is not None and nxt["type"] == 0 and int(nxt["op"]["target"]) == lpos
                        and not (nxt["op"]["u"][2] == 0 and nxt["op"]["u"][3] == 0
                                 and nxt["op"]["u"][4] == 0 and nxt["op"]["u"][5] == 0)):
                    gate = nxt
                dist.barrier()  # the partner's earlier work on its shard is done
                _xchg_role(oracle, shards, L, lpos, rank & ~bit, rank | bit, 1 if rank & bit else 0, gate)
                dist.barrier()  # both halves written before anyone goes on
                if gate is not None:
                    fused += 1
                    i += 1
            elif st["type"] == 3:
                mask, pos = multi_geometry(st)
                dist.barrier()
                _mxchg_role(shards, L, mask, pos, rank)
                dist.barrier()
            else:
                run_local_steps(oracle, L, shards[rank], rank, [st])
            i += 1
        dist.barrier()
        if rank == 0:
            got = np.concatenate(shards)
            want = oracle.simulate(n, gate_array(c))
            q.put((bool(np.array_equal(got, want)), fused))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,batch", [(2, 1), (4, 1), (4, 4)])
def test_gloo_peer_exchange_protocol_bit_identical(world, batch):
    import torch
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    for fn, args in [("u3_ladder_circuit", (10, 3, 5)), ("random_circuit", (8, 160, 4)),
                     ("haar_sweep_circuit", (9, 3))]:
        n = args[0]
        L = n - int(np.log2(world))
        tensors = [torch.zeros(2 << L, dtype=torch.float64).share_memory_() for _ in range(world)]
        tensors[0][0] = 1.0
        port = _free_port()
        procs = [ctx.Process(target=_peer_worker, args=(r, world, port, fn, args, tensors, q, batch))
                 for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(120)
            assert p.exitcode == 0
        ok, fused = q.get(timeout=10)
        assert ok, (fn, world)
        assert fused > 0 or batch > 1, (fn, world)


# --- property test: random circuits, shard counts and batching ------------------------
from hypothesis import given, settings, strategies as hs  # noqa: E402


@settings(max_examples=40, deadline=None)
@given(n=hs.integers(4, 9), g=hs.integers(1, 3), depth=hs.integers(1, 120), seed=hs.integers(0, 2**32 - 1),
       batch=hs.sampled_from([1, 2, 4]))
def test_schedule_property_random_circuits(qv, oracle, n, g, depth, seed, batch):
    """Any seeded random circuit (the reference's generator), any shard count
    with n >= g + 2, pairwise or batched exchanges: executing the schedule on
    CPU shards reproduces the oracle bit for bit, and the canonical restore
    leaves the qubit map at the identity."""
    if n < g + 2:
        return
    c = qv.random_circuit(n, depth, seed)
    steps = schedule(qv, c, 1 << g, canonicalize=True, batch=batch)
    want = oracle.simulate(n, gate_array(c))
    assert np.array_equal(emulate(oracle, n, 1 << g, steps), want)

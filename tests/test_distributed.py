"""Multi-rank host logic on CPU (gloo, world size 2 and 3): the summary exchange of
paper_1905_13415_b200/distributed.py composes per-range state-transition vectors and
record/column counts into each rank's entry context (the streaming context carry of
P:600-609).  Each rank's local summaries come from the oracle's sequential trace here (no GPU), and
the exchanged context must equal the sequential parser's state at the range boundary."""
import os
import random
import socket

import pytest
import torch.multiprocessing as mp

import oracle
from oracle import primitives as P
from paper_1905_13415_b200 import dialects

NONE = 0xFFFFFFFFFFFFFFFF
F_ABS, F_HD, F_IC, F_PC, F_PRE = 1, 2, 4, 8, 16


def seg_from_kinds(kinds, base):
    """Segment summary of a byte range from its per-byte emission kinds (test-side restatement of
    SURVEY §8a S5: records, delimiters, abs/rel column offset, open-field carries)."""
    from paper_1905_13415_b200 import _lib
    rec = sum(1 for k in kinds if k == 3)
    nd = sum(1 for k in kinds if k in (2, 3))
    last_rec = max((i for i, k in enumerate(kinds) if k == 3), default=None)
    last_d = max((i for i, k in enumerate(kinds) if k in (2, 3)), default=None)
    flags = 0
    if last_rec is not None:
        flags |= F_ABS
        col = sum(1 for k in kinds[last_rec + 1:] if k in (2, 3))
    else:
        col = nd
    if last_d is not None:
        flags |= F_HD
    open_part = list(enumerate(kinds))[(last_d + 1) if last_d is not None else 0:]
    data = [i for i, k in open_part if k == 0]
    ctrl = [i for i, k in open_part if k == 1]
    if data:
        fd, ld = data[0], data[-1]
        if any(c < fd for c in ctrl):
            flags |= F_PRE
        if any(c > ld for c in ctrl):
            flags |= F_PC
        if any(fd < c < ld for c in ctrl):
            flags |= F_IC
        fdg, ldg = base + fd, base + ld
    else:
        fdg = ldg = NONE
        if ctrl:
            flags |= F_PRE
    return _lib.Counts_t(rec, nd, fdg, ldg, col, flags, NONE)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, data, cuts, dialect, C, q):
    import torch.distributed as dist
    import paper_1905_13415_b200 as parpa
    from paper_1905_13415_b200 import distributed as pdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        t = dialects.get(dialect)
        dfa = parpa.Dfa.from_tables(t)
        lo, hi = cuts[rank], cuts[rank + 1]
        full = oracle.parse(dialect, data, C, trace=True)
        local_tau = P.tau(t.transition, t.group_of_byte, data[lo:hi])

        def count_fn(entry):
            assert entry == full.trace_state[lo] if lo < len(data) else True
            return seg_from_kinds(full.trace_kind[lo:hi].tolist(), lo)

        e, prefix, _ = pdist.exchange(dfa, local_tau, count_fn)
        # expected context at the boundary, from the sequential parse
        kinds = full.trace_kind[:lo].tolist()
        exp_state = full.trace_state[lo] if lo < len(data) else full.final_state
        exp = seg_from_kinds(kinds, 0)
        q.put((rank, e == exp_state, prefix.records == exp.records, prefix.fields == exp.fields,
               prefix.column == exp.column, prefix.open_first == exp.open_first,
               prefix.open_last == exp.open_last, (prefix.flags & 0x1C) == (exp.flags & 0x1C)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,dialect", [(2, "csv"), (3, "csv"), (2, "clf")])
def test_exchange_gives_sequential_context(world, dialect):
    import datagen
    wl = {"csv": "cfg1", "clf": "clf"}[dialect]
    data, _ = datagen.generate(wl, 60_000)
    data = bytes(data)
    rng = random.Random(world)
    inner = sorted(rng.sample(range(1, len(data) - 1), world - 1))
    cuts = [0] + inner + [len(data)]
    C = datagen.WORKLOADS[wl].C
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, data, cuts, dialect, C, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in sorted(results):
        assert all(r[1:]), r


def test_seg_helper_matches_fig_parser_two():
    # fig:parser_two: "a,b" rel(1); ",c\nd" abs(0); ",e\n" abs(0)
    r = oracle.parse("csv", b"a,b,c\nd,e\n", 3, trace=True)
    k = r.trace_kind.tolist()
    assert seg_from_kinds(k[0:3], 0).column == 1 and not seg_from_kinds(k[0:3], 0).flags & F_ABS
    s = seg_from_kinds(k[3:7], 3)
    assert s.column == 0 and s.flags & F_ABS and s.records == 1


# ---- the cross-rank halo (distributed.halo_plan / halo_exchange) ------------------------------------
def test_halo_plan_cases():
    from paper_1905_13415_b200.distributed import NONE64, halo_plan
    bases, lens = [0, 1000, 2000, 3000], [1000, 1000, 1000, 500]
    # rank 1: field from 970 (chunk 960 of rank 0); rank 2: nothing open; rank 3: field from 1500 (chunk
    # 1448 = 1000 + 7 * 64 of rank 1, two ranks); chunk boundaries are relative to the owning rank
    p = halo_plan(bases, lens, [NONE64, 970, NONE64, 1500])
    assert p == {1: (960, 0, [(0, 960, 1000)]), 3: (1448, 1, [(1, 1448, 2000), (2, 2000, 3000)])}
    # a field starting exactly at a rank boundary needs no halo
    assert halo_plan(bases, lens, [NONE64, 1000, 2000 - 64, NONE64]) == {2: (1896, 1, [(1, 1896, 2000)])}
    # beyond the cap: no halo (the device reports a straddling typed field as unsupported)
    assert halo_plan(bases, lens, [NONE64, NONE64, NONE64, 10], max_bytes=2000) == {}
    # the pieces always tile [h, base_g)
    import random
    rng = random.Random(5)
    for _ in range(200):
        G = rng.randint(2, 6)
        lens = [rng.randint(1, 300) for _ in range(G)]
        bases = [sum(lens[:i]) for i in range(G)]
        of = [NONE64] + [rng.choice([NONE64, rng.randrange(0, bases[g] + 1)]) for g in range(1, G)]
        for g, (h, r0, pieces) in halo_plan(bases, lens, of, chunk=16).items():
            assert pieces[0][1] == h and pieces[-1][2] == bases[g] and bases[r0] <= of[g] < bases[g]
            assert (h - bases[r0]) % 16 == 0 and h <= of[g] < h + 16
            assert all(pieces[i][2] == pieces[i + 1][1] for i in range(len(pieces) - 1))


class _TracePlan:
    """Stands in for a RangePlan: the state before a byte from the oracle's sequential trace."""
    def __init__(self, trace_state):
        self.trace_state = trace_state

    def state_at(self, pos):
        return int(self.trace_state[pos])


def _halo_worker(rank, world, port, data, cuts, q):
    import torch
    import torch.distributed as dist
    from paper_1905_13415_b200 import distributed as pdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        full = oracle.parse("csv", data, 4, trace=True)
        kinds = full.trace_kind.tolist()
        bases, lens = cuts[:-1], [cuts[i + 1] - cuts[i] for i in range(world)]
        open_first = [seg_from_kinds(kinds[:b], 0).open_first if b else pdist.NONE64 for b in bases]
        hplan = pdist.halo_plan(bases, lens, open_first)
        local = \
            torch.tensor(list(data[cuts[rank]:cuts[rank + 1]]), dtype=torch.uint8)
        left, state = pdist.halo_exchange(_TracePlan(full.trace_state), local, rank, bases, hplan)
        if rank in hplan:
            h = hplan[rank][0]
            ok = bytes(left.tolist()) == data[h:cuts[rank]] and state == int(full.trace_state[h])
        else:
            ok = left is None and state is None
        q.put((rank, ok, rank in hplan))
    finally:
        dist.destroy_process_group()


def test_halo_exchange_gloo_world3():
    """Ranks cut inside long quoted fields (one spanning a whole rank): each receives exactly the bytes
    from the chunk boundary before its straddling field's first DATA byte, with the DFA state there."""
    rng = random.Random(3)
    rows = []
    for i in range(120):
        long = '"' + "".join(rng.choice('ab ,\n""') for _ in range(rng.randint(50, 400))) + '"'
        rows.append(f"{i},{long},{rng.randint(0, 999)}\n")
    rows.insert(60, "7," + '"' + "x" * 5000 + '"' + ",1\n")
    data = "".join(rows).encode()
    mid = data.index(b"x" * 5000)
    cuts = [0, mid + 100, mid + 3000, len(data)]          # ranks 1 and 2 start inside the 5000-byte field
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, 3, port, data, cuts, q)) for r in range(3)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(3))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(r[1] for r in res), res
    assert res[1][2] and res[2][2]                          # both later ranks needed a halo

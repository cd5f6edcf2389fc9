"""Multi-GPU sharded parse: contiguous byte ranges, one summary exchange.

Each rank holds one contiguous byte range [base, base+len) of the logical input (NOT record
aligned).  The context of a range is the composition of the summaries of all ranges before it —
the paper's streaming context carry (seed state, column and record offset) applied
across GPUs:

  1. τ_g = parpa_summarize(range g)                 (state-transition vector of the range)
     allgather τ  ->  entry state e_g = (τ_0 ∘ … ∘ τ_{g-1})[start]
  2. counts_g = parpa_count(range g, e_g)           (records, fields, abs/rel column, open-field carries)
     allgather counts  ->  prefix_g = counts_0 ⊕ … ⊕ counts_{g-1}
  3. parpa_parse_range(range g, e_g, prefix_g)      -> columns stay sharded; row r of rank g is global
                                                        record prefix_g.records + r.

The two allgathers move 16 B and 48 B per rank (torch.distributed, NCCL over NVLink on GPUs, gloo
on CPU).  The composition itself runs on the host through the C ABI (parpa_compose_tau,
parpa_compose_counts) — no device work, so this module's exchange logic is testable on CPU.
"""
from __future__ import annotations

import ctypes

from . import _lib

TAU_BYTES = ctypes.sizeof(_lib.Tau_t)
COUNTS_BYTES = ctypes.sizeof(_lib.Counts_t)


def _allgather_bytes(payload: bytes, group=None, device=None):
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    t = torch.frombuffer(bytearray(payload), dtype=torch.uint8)
    if device is not None:
        t = t.to(device)
    out = torch.empty(world * len(payload), dtype=torch.uint8, device=t.device)
    dist.all_gather_into_tensor(out, t, group=group)
    raw = out.cpu().numpy().tobytes()
    return [raw[i * len(payload):(i + 1) * len(payload)] for i in range(world)]


def tau_to_bytes(tau: list) -> bytes:
    t = _lib.Tau_t()
    for i in range(16):
        t.tau[i] = tau[i] if i < len(tau) else 0xFF
    return bytes(t)


def tau_from_bytes(b: bytes, nstates: int) -> list:
    return list(_lib.Tau_t.from_buffer_copy(b).tau[:nstates])


def entry_state(dfa, taus: list, rank: int) -> int:
    """(τ_0 ∘ … ∘ τ_{rank-1})[start] by host composition through the C ABI."""
    from . import compose_tau
    acc = list(range(dfa.num_states))
    for g in range(rank):
        acc = compose_tau(dfa, acc, taus[g])
    return acc[dfa.start]


def prefix_counts(counts: list, rank: int):
    from . import compose_counts, identity_counts
    acc = identity_counts()
    for g in range(rank):
        acc = compose_counts(acc, counts[g])
    return acc


def exchange(dfa, local_tau: list, count_fn, group=None, device=None):
    """Two-step exchange.  ``count_fn(entry_state) -> Counts_t`` runs the range's count pass.
    Returns (entry_state, prefix Counts_t, all Counts_t)."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    taus = [tau_from_bytes(b, dfa.num_states) for b in _allgather_bytes(tau_to_bytes(local_tau), group, device)]
    e = entry_state(dfa, taus, rank)
    local = count_fn(e)
    counts = [_lib.Counts_t.from_buffer_copy(b) for b in _allgather_bytes(bytes(local), group, device)]
    return e, prefix_counts(counts, rank), counts


NONE64 = (1 << 64) - 1
CHUNK_BYTES = 64                       # parpa_chunk_bytes(): the halo starts on a chunk boundary of its owner
HALO_MAX = 256 << 20                   # larger halos are not sent (a typed field that long: EUNSUPPORTED)


def halo_plan(bases, lens, open_first, chunk=CHUNK_BYTES, max_bytes=HALO_MAX):
    """The cross-rank halo (the multi-GPU analogue of the paper's partition carry-over).

    Rank g needs the bytes of the field left open at its start that lie before it: from h_g = the chunk
    boundary (of the rank owning it) at or before the field's first DATA byte open_first[g] up to base_g,
    plus the DFA state at h_g (so that inner control bytes can be re-simulated).  The ranges are
    contiguous (base_{r+1} = base_r + len_r).  Returns {g: (h_g, r0, [(r, lo, hi), ...])}: r0 owns h_g and
    supplies the state; the pieces, in rank order, cover [h_g, base_g).  Pure (testable on the host)."""
    G = len(bases)
    plan = {}
    for g in range(1, G):
        fd = open_first[g]
        if fd == NONE64 or fd >= bases[g]:
            continue
        r0 = max(r for r in range(g) if bases[r] <= fd)
        h = bases[r0] + ((fd - bases[r0]) // chunk) * chunk
        if bases[g] - h > max_bytes:
            continue
        pieces = []
        for r in range(r0, g):
            lo, hi = max(h, bases[r]), min(bases[r] + lens[r], bases[g])
            if lo < hi:
                pieces.append((r, lo, hi))
        plan[g] = (h, r0, pieces)
    return plan


def halo_exchange(plan_obj, data, rank, bases, hplan, group=None, device=None):
    """One all_to_all (NCCL over NVLink on GPUs): every rank sends the pieces of its range that later
    ranks need, the owner of h_g prefixing its piece with the DFA state at h_g.  Returns (left tensor on
    data's device or None, left DFA state or None)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if not hplan:                                       # the same on every rank: nobody needs a halo
        return None, None
    dev = device if device is not None else data.device
    send_parts, in_splits = [], [0] * world
    for g in range(world):
        if g not in hplan:
            continue
        h, r0, pieces = hplan[g]
        for r, lo, hi in pieces:
            if r != rank:
                continue
            part = data[lo - bases[rank]:hi - bases[rank]].to(dev)
            if r == r0:
                st = torch.tensor([plan_obj.state_at(h)], dtype=torch.uint8, device=dev)
                part = torch.cat([st, part])
            send_parts.append(part)
            in_splits[g] = part.numel()
    out_splits = [0] * world
    if rank in hplan:
        h, r0, pieces = hplan[rank]
        for r, lo, hi in pieces:
            out_splits[r] = (hi - lo) + (1 if r == r0 else 0)
    inp = torch.cat(send_parts) if send_parts else torch.empty(0, dtype=torch.uint8, device=dev)
    out = torch.empty(sum(out_splits), dtype=torch.uint8, device=dev)
    dist.all_to_all_single(out, inp, out_splits, in_splits, group=group)
    if rank not in hplan:
        return None, None
    state = int(out[0].item())
    return out[1:].to(data.device), state


def parse_sharded(dfa, schema, data, base: int, columns, capacity: int, stats_tensor, left=None,
                  is_last: bool | None = None, group=None, stream=None, exchange_device=None):
    """Parse this rank's range after the summary exchange.  data / left: CUDA uint8 tensors.
    Every pass runs once per rank: S1-S3 (range_begin) -> allgather τ -> S4-S5 from the entry
    state (range_count) -> allgather counts -> S6-S7 with the ⊕-prefix (range_emit).  ``is_last``
    (the range ends the input, so the end-of-input action applies) defaults to "this is the group's
    last rank".  With ``left=None`` the left context is exchanged between the ranks (halo_plan /
    halo_exchange: exactly the bytes of the field straddling each boundary, with the DFA state at their
    start); an explicit ``left`` is used as given (state unknown)."""
    import struct
    import torch.distributed as dist
    from . import RangePlan
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if is_last is None:
        is_last = rank == world - 1
    dev = exchange_device if exchange_device is not None else data.device
    plan = RangePlan(dfa, data, base, stream)
    try:
        e, prefix, counts = exchange(dfa, plan.tau, plan.count, group, dev)
        left_state = None
        if left is None and world > 1:
            bl = [struct.unpack("<QQ", b) for b in _allgather_bytes(struct.pack("<QQ", int(base), data.numel()),
                                                                     group, dev)]
            bases, lens = [x[0] for x in bl], [x[1] for x in bl]
            open_first = [prefix_counts(counts, g).open_first for g in range(world)]
            left, left_state = halo_exchange(plan, data, rank, bases, halo_plan(bases, lens, open_first), group, dev)
        plan.emit(schema, prefix, columns, capacity, stats_tensor, left=left, is_last=is_last, left_state=left_state)
    finally:
        plan.close()
    return e, prefix

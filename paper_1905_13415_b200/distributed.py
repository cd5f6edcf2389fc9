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


def parse_sharded(dfa, schema, data, base: int, columns, capacity: int, stats_tensor, left=None,
                  is_last: bool | None = None, group=None, stream=None, exchange_device=None):
    """Parse this rank's range after the summary exchange.  data / left: CUDA uint8 tensors.
    Every pass runs once per rank: S1-S3 (range_begin) -> allgather τ -> S4-S5 from the entry
    state (range_count) -> allgather counts -> S6-S7 with the ⊕-prefix (range_emit).  ``is_last``
    (the range ends the input, so the end-of-input action applies) defaults to "this is the group's
    last rank"."""
    import torch.distributed as dist
    from . import RangePlan
    if is_last is None:
        is_last = dist.get_rank(group) == dist.get_world_size(group) - 1
    plan = RangePlan(dfa, data, base, stream)
    try:
        e, prefix, _ = exchange(dfa, plan.tau, plan.count, group,
                                exchange_device if exchange_device is not None else data.device)
        plan.emit(schema, prefix, columns, capacity, stats_tensor, left=left, is_last=is_last)
    finally:
        plan.close()
    return e, prefix

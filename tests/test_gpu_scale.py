"""GPU parity at scale.

1. Element-wise parity (all three API paths) on inputs that span several blocks of the two decoupled
   look-back scans (one scan block = 2048 warp tiles = 4 MB), so that block aggregates, inclusive
   prefixes and the look-back windows are all exercised against the oracle.
2. The bench configuration itself (BASELINE configs[1]-[3] at full size, parse_into, the launch
   configuration bench.py times): sampled records are checked against the oracle run on the
   generator's text of that record (offsets relative to the record, lengths, values, valid flags),
   the record's bytes are found at the offsets the GPU reports, and the whole columns are checked
   against the generator's ground truth (record count, wrapping sum and null count of every int64
   column: pin G1)."""
import os
import random

import numpy as np
import pytest

import datagen
import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import paper_1905_13415_b200 as parpa  # noqa: E402
from tests.test_gpu_parity import run_all_paths  # noqa: E402


@pytest.mark.parametrize("name,nbytes", [("cfg1", 18_000_000), ("yelp", 22_000_000), ("clf", 21_000_000),
                                         ("taxi", 13_000_000)])
def test_multi_scan_block_full_compare(name, nbytes):
    w = datagen.WORKLOADS[name]
    data, g = datagen.generate(name, nbytes)
    assert g.nbytes > 3 * parpa.tile_bytes() * 2048
    ora = run_all_paths(w.dialect, data, w.types, label=f"{name}-{nbytes}")
    assert ora.R == g.records


def _wrap_sum(a):
    return int(np.sum(a.astype(np.uint64), dtype=np.uint64).astype(np.int64))


@pytest.mark.parametrize("name", ["taxi", "yelp", "clf"])
def test_full_size_sampled_against_oracle(name):
    if os.environ.get("PARPA_SKIP_FULL"):
        pytest.skip("PARPA_SKIP_FULL set")
    w = datagen.WORKLOADS[name]
    free, _ = torch.cuda.mem_get_info()
    if free < 60e9:
        pytest.skip("needs a B200-sized device")
    buf = torch.empty(w.target_bytes, dtype=torch.uint8, pin_memory=True)
    g = datagen.fill(name, buf.data_ptr(), w.target_bytes)
    host = buf[:g.nbytes].numpy()
    d = buf[:g.nbytes].to("cuda")
    dfa = parpa.Dfa.dialect(w.dialect)
    schema = parpa.Schema(list(w.types))
    cap = g.records + 2
    cols = parpa.alloc_columns(schema, cap)
    st = parpa.new_stats_tensor()
    parpa.parse_into(dfa, schema, d, cols, cap, st)
    torch.cuda.synchronize()
    s = parpa.stats_from_tensor(st)
    assert s["status"] == 0 and s["records"] == g.records, (s, g.records)
    assert s["missing_records"] == 0 and s["extra_fields"] == 0
    # whole-column ground truth: int64 sums and nulls (generator, pin G1)
    ints = [c for c, t in enumerate(w.types) if t == datagen.INT64]
    R = g.records
    for j, c in enumerate(ints):
        v = cols[c].value[:R].view(torch.int64)
        ok = cols[c].valid[:R].bool()
        assert int((~ok).sum().item()) == g.int_nulls[j], (name, c)
        s64 = int(torch.where(ok, v, torch.zeros_like(v)).sum().item())   # torch sums int64 with wrap-around
        assert s64 == g.int_sums[j], (name, c, s64, g.int_sums[j])
    # sampled records against the oracle on the record's own text
    rng = random.Random(7)
    idx = sorted(set([0, 1, R - 1] + rng.sample(range(R), 1500)))
    it = torch.tensor(idx, dtype=torch.int64, device="cuda")
    off = [cols[c].offset.view(torch.int64)[it].cpu().numpy() for c in range(w.C)]
    ln = [cols[c].length.view(torch.int32)[it].cpu().numpy().view(np.uint32) for c in range(w.C)]
    val = [cols[c].value.view(torch.int64)[it].cpu().numpy() if w.types[c] != datagen.SPAN else None
           for c in range(w.C)]
    ok = [cols[c].valid[it].cpu().numpy() if w.types[c] != datagen.SPAN else None for c in range(w.C)]
    for n, i in enumerate(idx):
        rec = datagen.record(name, i)
        o = oracle.parse(w.dialect, rec, w.C, list(w.types))
        assert o.status == 0 and o.R == 1, (name, i)
        start = int(off[0][n]) - int(o.offset[0][0])
        assert bytes(host[start:start + len(rec)]) == rec, (name, i, start)
        for c in range(w.C):
            assert int(off[c][n]) == start + int(o.offset[c][0]), (name, i, c)
            assert int(ln[c][n]) == int(o.length[c][0]), (name, i, c)
            if w.types[c] != datagen.SPAN:
                assert int(ok[c][n]) == int(o.valid[c][0]), (name, i, c)
                assert int(val[c][n]) == int(o.value[c][0]), (name, i, c, int(val[c][n]), int(o.value[c][0]))
    del cols, d
    torch.cuda.empty_cache()

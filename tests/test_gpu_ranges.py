"""GPU: range summaries and sharded parsing (the multi-GPU path) on one GPU with "virtual ranks".

The input is cut at arbitrary byte positions (inside quoted fields, on delimiters, at ±1 of them);
each range is summarised on the GPU (parpa_summarize / parpa_count), the summaries are composed on
the host exactly as distributed.exchange does across ranks, every range is parsed with
parpa_parse_range, and the concatenated rows must equal the oracle's single-shot parse."""
import random

import numpy as np
import pytest

import datagen
import oracle
from tests.gpu_helpers import to_np

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import paper_1905_13415_b200 as parpa  # noqa: E402
from paper_1905_13415_b200 import distributed as pdist  # noqa: E402


def dev(a):
    t = torch.empty(max(len(a), 1) + 16, dtype=torch.uint8, device="cuda")
    if len(a):
        t[:len(a)].copy_(torch.from_numpy(np.frombuffer(bytes(a), np.uint8).copy()))
    return t[:len(a)]


def sharded_parse(dialect, data, types, cuts, left_bytes=4096, staged=False, halo=False):
    """Parse every range as its own "rank" and assemble the global columns.  Columns stay sharded
    (SURVEY §8e): the record straddling cut g has its columns < col(g) on rank g-1 (local row
    R_local) and the rest on rank g (local row 0).  staged=True uses the range plan
    (parpa_range_begin / _count / _emit: every pass once), else summarize / count / parse_range."""
    dfa = parpa.Dfa.dialect(dialect)
    schema = parpa.Schema(list(types))
    G = len(cuts) - 1
    taus, counts = [], []
    plans = [parpa.RangePlan(dfa, dev(data[cuts[g]:cuts[g + 1]]), cuts[g]) for g in range(G)] if staged else None
    for g in range(G):
        taus.append(plans[g].tau if staged else parpa.summarize(dfa, dev(data[cuts[g]:cuts[g + 1]])))
    for g in range(G):
        e = pdist.entry_state(dfa, taus, g)
        if staged:
            c = plans[g].count(e)
        else:
            c, tau2 = parpa.count(dfa, dev(data[cuts[g]:cuts[g + 1]]), cuts[g], e)
            assert tau2 == taus[g]
        counts.append(c)
    C = len(types)
    out = [[[] for _ in range(4)] for _ in range(C)]
    hplan = {}
    if halo:                     # the exact halo of distributed.halo_plan, state from the owner's plan
        assert staged
        bases, lens = cuts[:-1], [cuts[g + 1] - cuts[g] for g in range(G)]
        open_first = [pdist.prefix_counts(counts, g).open_first for g in range(G)]
        hplan = pdist.halo_plan(bases, lens, open_first)
    for g in range(G):
        e = pdist.entry_state(dfa, taus, g)
        prefix = pdist.prefix_counts(counts, g)
        after = pdist.prefix_counts(counts, g + 1)
        lo, hi = cuts[g], cuts[g + 1]
        cap = (hi - lo) + 2
        cols = parpa.alloc_columns(schema, cap)
        st = parpa.new_stats_tensor()
        left = dev(data[max(0, lo - left_bytes):lo]) if lo else None
        last = g == G - 1
        left_state = None
        if halo:
            left = None
            if g in hplan:
                h, r0, _ = hplan[g]
                left, left_state = dev(data[h:lo]), plans[r0].state_at(h)
        if staged:
            plans[g].emit(schema, prefix, cols, cap, st, left=left, is_last=last, left_state=left_state)
        else:
            parpa.parse_range(dfa, schema, dev(data[lo:hi]), e, lo, prefix, cols, cap, st, left=left, is_last=last)
        s = parpa.stats_from_tensor(st)
        assert s["status"] in (0, parpa.ECOLUMNS), s
        n = s["records"]
        c_in, c_out = prefix.column, after.column
        for c in range(C):
            rows = list(range(n + (0 if last else 1)))
            keep = []
            for r in rows:
                ok = True
                if r == 0 and c < c_in:
                    ok = False                 # closed on an earlier rank
                if r == n and not last and c >= c_out:
                    ok = False                 # closed on a later rank
                if ok:
                    keep.append(r)
            arrs = [cols[c].offset, cols[c].length, cols[c].value, cols[c].valid]
            views = [np.uint64, np.uint32, np.int64, None]
            for i in range(4):
                if arrs[i] is None:
                    continue
                a = to_np(arrs[i])
                a = a.view(views[i]) if views[i] is not None else a
                out[c][i].append(a[keep])
    return [tuple(np.concatenate(x[i]) if x[i] else None for i in range(4)) for x in out]


@pytest.mark.parametrize("staged", [False, True])
@pytest.mark.parametrize("name,G,seed", [("cfg1", 2, 0), ("cfg1", 5, 1), ("yelp", 3, 2), ("clf", 4, 3),
                                         ("taxi", 3, 4)])
def test_virtual_ranks_equal_single_shot(name, G, seed, staged):
    w = datagen.WORKLOADS[name]
    data, _ = datagen.generate(name, 1_500_000)
    data = bytes(data)
    ora = oracle.parse(w.dialect, data, w.C, list(w.types))
    rng = random.Random(seed)
    inner = sorted(rng.sample(range(1, len(data) - 1), G - 1))
    # nudge one cut onto a delimiter and one just after, and keep 16-byte alignment of nothing in particular
    cuts = [0] + inner + [len(data)]
    cols = sharded_parse(w.dialect, data, w.types, cuts, staged=staged)
    for c, t in enumerate(w.types):
        off, ln, val, ok = cols[c]
        assert np.array_equal(off, ora.offset[c]), (name, c)
        assert np.array_equal(ln, ora.length[c]), (name, c)
        if t != oracle.SPAN:
            assert np.array_equal(ok, ora.valid[c]), (name, c)
            assert np.array_equal(val, ora.value[c]), (name, c)


def test_cuts_at_delimiters_and_inside_quotes():
    data = b'1,"Hello, World\nHow are you?",3\n' * 400 + b'x,"a""b",7\n' * 300
    types = [oracle.SPAN, oracle.SPAN, oracle.INT64]
    ora = oracle.parse("csv", data, 3, types)
    special = [i for i in range(1, len(data) - 1) if data[i] in b',\n"']
    rng = random.Random(9)
    for trial in range(6):
        picks = sorted(set(rng.sample(special, 3) + [rng.choice(special) + 1]))
        cuts = [0] + picks + [len(data)]
        cols = sharded_parse("csv", data, types, cuts, staged=bool(trial & 1))
        for c in range(3):
            assert np.array_equal(cols[c][0], ora.offset[c])
            assert np.array_equal(cols[c][1], ora.length[c])
        assert np.array_equal(cols[2][2], ora.value[2])


@pytest.mark.parametrize("staged", [False, True])
def test_virtual_ranks_adversarial_plain(staged):
    """Ranges over CTRL-free data with giant fields and long numbers crossing the cuts (their leading bytes
    come from the left context), far more device-tier fields than the queue holds, ragged records."""
    from tests.gpu_helpers import adversarial_plain
    data, types = adversarial_plain(11, nrows=30000)
    ora = oracle.parse("csv", data, len(types), types)
    rng = random.Random(12)
    cuts = [0] + sorted(rng.sample(range(1, len(data) - 1), 4)) + [len(data)]
    cols = sharded_parse("csv", data, types, cuts, left_bytes=80000, staged=staged)
    for c, t in enumerate(types):
        off, ln, val, ok = cols[c]
        assert np.array_equal(off, ora.offset[c]), c
        assert np.array_equal(ln, ora.length[c]), c
        if t != oracle.SPAN:
            assert np.array_equal(ok, ora.valid[c]), c
            assert np.array_equal(val, ora.value[c]), c


def test_virtual_ranks_adversarial_clf():
    """Ranges over the adversarial CLF lines, cuts anywhere (inside brackets, quotes, escapes, comments)."""
    from tests.gpu_helpers import adversarial_clf
    data, types = adversarial_clf(3, nlines=20000)
    ora = oracle.parse("clf", data, len(types), types)
    rng = random.Random(13)
    cuts = [0] + sorted(rng.sample(range(1, len(data) - 1), 5)) + [len(data)]
    cols = sharded_parse("clf", data, types, cuts, staged=True)
    for c, t in enumerate(types):
        off, ln, val, ok = cols[c]
        assert np.array_equal(off, ora.offset[c]), c
        assert np.array_equal(ln, ora.length[c]), c
        if t != oracle.SPAN:
            assert np.array_equal(ok, ora.valid[c]), c
            assert np.array_equal(val, ora.value[c]), c


def test_range_plan_repeated_count_and_emit():
    """A range plan counted and emitted more than once: every repeat must return the same
    counts and columns as the first call and as the oracle (the control words and look-back flags are
    cleared per call)."""
    w = datagen.WORKLOADS["cfg1"]
    data, g = datagen.generate("cfg1", 300_000)
    ora = oracle.parse(w.dialect, data, w.C, list(w.types))
    dfa = parpa.Dfa.dialect(w.dialect)
    schema = parpa.Schema(list(w.types))
    plan = parpa.RangePlan(dfa, dev(data), 0)
    try:
        c1 = bytes(plan.count(dfa.start))
        c2 = bytes(plan.count(dfa.start))
        assert c1 == c2
        prefix = pdist.prefix_counts([], 0)
        for _ in range(3):
            cols = parpa.alloc_columns(schema, ora.R)
            st = parpa.new_stats_tensor()
            plan.emit(schema, prefix, cols, ora.R, st, is_last=True)
            s = parpa.stats_from_tensor(st)
            assert s["status"] == 0 and s["records"] == ora.R and s["missing_records"] == ora.n_missing, s
            for c, t in enumerate(w.types):
                assert np.array_equal(to_np(cols[c].offset).view(np.uint64)[:ora.R], ora.offset[c])
                assert np.array_equal(to_np(cols[c].length).view(np.uint32)[:ora.R], ora.length[c])
                if t != datagen.SPAN:
                    assert np.array_equal(to_np(cols[c].value).view(np.int64)[:ora.R], ora.value[c])
                    assert np.array_equal(to_np(cols[c].valid).view(np.uint8)[:ora.R], ora.valid[c])
    finally:
        plan.close()


@pytest.mark.parametrize("seed", [0, 1])
def test_virtual_ranks_exact_halo_long_and_inner_control_fields(seed):
    """The cross-rank halo (distributed.halo_plan): each range receives exactly the bytes of the field
    straddling its start, from the owner's chunk boundary, with the DFA state there.  Fields of 4-9 KB
    straddle the cuts: quoted numbers with "" inside (inner control bytes: the device tier re-simulates
    the halo from its state — before this, PARPA_EUNSUPPORTED), long floats and long quoted text."""
    rng = random.Random(seed)
    rows = []
    for i in range(3000):
        a = rng.randint(-999, 999)
        b = f"{rng.randint(0, 99999)}.{rng.randint(0, 999)}"
        t = '"' + "".join(rng.choice("abc ,\n") for _ in range(rng.randint(0, 60))) + '"'
        rows.append(f"{a},{b},{t}\n")
    giants = ['"1' + "2" * 4500 + '""' + "3" * 3000 + '"',       # typed, inner control byte: invalid
              "1" * 6000 + "." + "5" * 2000,                     # a 8 KB float: valid, device tier
              '"' + "7" * 5000 + '"']                            # a quoted 5 KB integer: invalid (overflow)
    pos = sorted(rng.sample(range(100, 2900), 6))
    for k, p in enumerate(pos):
        g = giants[k % 3]
        rows[p] = (f"{g},1.5,x\n" if k % 3 != 1 else f"3,{g},\"t\"\n")
    data = "".join(rows).encode()
    types = [oracle.INT64, oracle.FLOAT64, oracle.SPAN]
    ora = oracle.parse("csv", data, 3, types)
    assert ora.status == 0
    # cut inside the giant fields (and elsewhere)
    starts = [data.index(g.encode()) for g in giants if g.encode() in data]
    inner = sorted(set([s0 + 2500 for s0 in starts] + rng.sample(range(1, len(data) - 1), 2)))
    cuts = [0] + inner + [len(data)]
    cols = sharded_parse("csv", data, types, cuts, staged=True, halo=True)
    for c, t in enumerate(types):
        off, ln, val, ok = cols[c]
        assert np.array_equal(off, ora.offset[c]), c
        assert np.array_equal(ln, ora.length[c]), c
        if t != oracle.SPAN:
            assert np.array_equal(ok, ora.valid[c]), c
            assert np.array_equal(val, ora.value[c]), c


@pytest.mark.parametrize("big", [3000, 300_000])
def test_virtual_ranks_collab_numbers_across_cuts(big):
    """Long raw numbers (block tier >= 1 KB, device tier >= 256 KB) cut by a range boundary:
    the owner reads the leading digits from the exact halo; values and validity equal the oracle's."""
    rng = random.Random(big)
    rows = [f"{i},{i}.25,r\n" for i in range(2000)]
    z = "0" * big
    nums = [("i", z + "77"), ("f", "1" * big + "." + "25"), ("f", "0." + z + "5e" + str(big + 3)),
            ("i", "9" * big), ("f", z + "x")]
    pos = sorted(rng.sample(range(50, 1950), len(nums)))
    for (kind, s), p in zip(nums, pos):
        rows[p] = f"{s},0.5,i\n" if kind == "i" else f"4,{s},f\n"
    data = "".join(rows).encode()
    types = [oracle.INT64, oracle.FLOAT64, oracle.SPAN]
    ora = oracle.parse("csv", data, 3, types)
    starts = [data.index(s.encode()) for _, s in nums]
    inner = sorted(set(s0 + len(nums[k][1]) // 2 for k, s0 in enumerate(starts)))
    cuts = [0] + inner + [len(data)]
    cols = sharded_parse("csv", data, types, cuts, staged=True, halo=True)
    for c, t in enumerate(types):
        off, ln, val, ok = cols[c]
        assert np.array_equal(off, ora.offset[c]), c
        assert np.array_equal(ln, ora.length[c]), c
        if t != oracle.SPAN:
            assert np.array_equal(ok, ora.valid[c]), c
            assert np.array_equal(val, ora.value[c]), c

"""GPU: string materialisation from a plan (the chunk masks reused) in the paper's three CSS layouts
 and the CSS index generation, element by element against the oracle."""
import numpy as np
import pytest

import datagen
import oracle

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import paper_1905_13415_b200 as parpa  # noqa: E402


def dev(data):
    a = np.frombuffer(bytes(data), np.uint8)
    t = torch.empty(max(a.size, 1), dtype=torch.uint8, device="cuda")
    if a.size:
        t[:a.size].copy_(torch.from_numpy(a.copy()))
    return t[:a.size]


@pytest.mark.parametrize("name,cols,nbytes", [("cfg1", [0, 3, 5, 7], 1_500_000), ("yelp", [0, 7, 8], 6_000_000),
                                              ("clf", [2, 3, 4], 4_000_000), ("taxi", [1, 6], 3_000_000)])
def test_plan_css_layouts(name, cols, nbytes):
    w = datagen.WORKLOADS[name]
    data, g = datagen.generate(name, nbytes)
    d = dev(data)
    with parpa.Plan(parpa.Dfa.dialect(w.dialect), d) as plan:
        res = plan.emit(parpa.Schema(list(w.types)))
        R = res.records
        assert R == g.records
        for c in cols:
            for mode in (parpa.CSS_ARROW, parpa.CSS_INLINE, parpa.CSS_VECTOR):
                want = oracle.css(w.dialect, data, w.C, c, list(w.types), mode=mode, terminator=0x1F)
                got = plan.strings(res.columns[c], R, mode=mode, terminator=0x1F)
                assert np.array_equal(got[0].cpu().numpy(), want[0]), (name, c, mode)
                assert bytes(got[1].cpu().numpy()) == want[1], (name, c, mode)
                if mode == parpa.CSS_VECTOR:
                    assert bytes(got[2].cpu().numpy()) == want[2], (name, c)
                if mode != parpa.CSS_ARROW:
                    buf = got[1] if mode == parpa.CSS_INLINE else got[2]
                    idx = parpa.css_index(mode, buf, 0x1F).cpu().numpy()
                    ref = oracle.css_index(mode, want[1] if mode == parpa.CSS_INLINE else want[2], 0x1F)
                    assert np.array_equal(idx, ref), (name, c, mode)


def test_plan_strings_equal_one_shot_strings():
    """the plan path (masks reused) and the one-shot parpa_strings_* path (scan re-run) agree"""
    w = datagen.WORKLOADS["yelp"]
    data, _ = datagen.generate("yelp", 3_000_000)
    d = dev(data)
    dfa = parpa.Dfa.dialect("csv")
    with parpa.Plan(dfa, d) as plan:
        res = plan.emit(parpa.Schema(list(w.types)))
        for c in (0, 7):
            o1, b1 = plan.strings(res.columns[c], res.records)
            o2, b2 = parpa.strings(dfa, d, res.columns[c], res.records)
            assert torch.equal(o1, o2) and torch.equal(b1, b2)


def test_inline_terminator_clash_reported():
    """the inline-terminated layout needs a terminator absent from the CSS"""
    data = b"a,b\nx\x1fy,z\n" * 100
    d = dev(data)
    with parpa.Plan(parpa.Dfa.dialect("csv"), d) as plan:
        res = plan.emit(parpa.Schema([oracle.SPAN, oracle.SPAN]))
        with pytest.raises(parpa.ParpaError):
            plan.strings(res.columns[0], res.records, mode=parpa.CSS_INLINE, terminator=0x1F)
        offs, buf = plan.strings(res.columns[0], res.records, mode=parpa.CSS_INLINE, terminator=0x1E)
        assert bytes(buf.cpu().numpy()) == b"a\x1ex\x1fy\x1e" * 100


def test_result_accessors_and_allocator_hook():
    """parpa_result_records / parpa_result_status, and result buffers from a caller-set
    allocator (torch's caching allocator through parpa_set_allocator)"""
    import ctypes
    from paper_1905_13415_b200 import _lib
    w = datagen.WORKLOADS["cfg1"]
    data, g = datagen.generate("cfg1", 500_000)
    d = dev(data)
    dfa = parpa.Dfa.dialect("csv")
    schema = parpa.Schema(list(w.types))
    ora = oracle.parse("csv", data, w.C, list(w.types))
    before = torch.cuda.memory_allocated()
    parpa.use_torch_allocator(True)
    try:
        res = parpa.parse_c_owned(dfa, schema, d)
        assert res.records == ora.R
        assert np.array_equal(res.columns[1].value.cpu().numpy().view(np.int64)[:ora.R], ora.value[1])
        L = _lib.load()
        r = ctypes.c_void_p()
        sch = schema.struct()
        assert L.parpa_parse(dfa.handle, ctypes.byref(sch), ctypes.c_void_p(d.data_ptr()), d.numel(), None,
                             ctypes.byref(r)) == 0
        assert torch.cuda.memory_allocated() > before            # the buffers came from torch
        R, st, fi, nm, ne = ctypes.c_uint64(), ctypes.c_int(), ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        assert L.parpa_result_records(r, ctypes.byref(R)) == 0 and R.value == ora.R
        assert L.parpa_result_status(r, ctypes.byref(st), ctypes.byref(fi), ctypes.byref(nm), ctypes.byref(ne)) == 0
        assert st.value == 0 and nm.value == ora.n_missing and ne.value == ora.n_extra
        L.parpa_result_free(r)
        torch.cuda.synchronize()
    finally:
        parpa.use_torch_allocator(False)


def test_error_paths_of_the_round2_entry_points():
    """EINVAL / ENOMEM of the plan-strings, CSS-index, workspace and allocator entry points (include/parpa.h)"""
    import ctypes
    from paper_1905_13415_b200 import _lib
    L = _lib.load()
    data = b"1,a\n2,b\n" * 1000
    d = dev(data)
    with parpa.Plan(parpa.Dfa.dialect("csv"), d) as plan:
        res = plan.emit(parpa.Schema([oracle.INT64, oracle.SPAN]))
        col = res.columns[1].struct()
        offs = torch.empty(res.records + 1, dtype=torch.int64, device="cuda")
        total = ctypes.c_uint64()
        assert L.parpa_plan_strings_size(plan._plan, ctypes.byref(col), res.records, 3, ctypes.c_void_p(offs.data_ptr()),
                                         ctypes.byref(total), None) == parpa.EINVAL          # mode > 2
        assert L.parpa_plan_strings_copy(plan._plan, ctypes.byref(col), res.records, parpa.CSS_VECTOR, 0x1F,
                                         ctypes.c_void_p(offs.data_ptr()), ctypes.c_void_p(offs.data_ptr()), None,
                                         None) == parpa.EINVAL                               # VECTOR without aux
    cnt = ctypes.c_uint64(7)
    assert L.parpa_css_index(parpa.CSS_INLINE, 0x1F, None, None, 0, None, ctypes.byref(cnt), None) == 0 and cnt.value == 0
    assert L.parpa_css_index(parpa.CSS_ARROW, 0x1F, None, None, 0, None, ctypes.byref(cnt), None) == parpa.EINVAL
    ws = parpa.Workspace(1 << 20)
    mis = torch.empty(len(data) + 16, dtype=torch.uint8, device="cuda")[1:1 + len(data)]
    mis.copy_(d)
    schema = parpa.Schema([oracle.INT64, oracle.SPAN])
    cols = parpa.alloc_columns(schema, 2100)
    with pytest.raises(parpa.ParpaError):                                                  # misaligned input
        parpa.parse_into(parpa.Dfa.dialect("csv"), schema, mis, cols, 2100, parpa.new_stats_tensor(), workspace=ws)
    ws.close()
    # an allocator that fails: parpa_parse reports ENOMEM and leaves nothing behind
    fail = parpa._ALLOC_FN(lambda n, s, c: None)
    free = parpa._FREE_FN(lambda p, s, c: None)
    assert L.parpa_set_allocator(ctypes.cast(fail, ctypes.c_void_p), None, None) == parpa.EINVAL   # one of two NULL
    assert L.parpa_set_allocator(ctypes.cast(fail, ctypes.c_void_p), ctypes.cast(free, ctypes.c_void_p), None) == 0
    try:
        r = ctypes.c_void_p()
        sch = schema.struct()
        dfa_csv = parpa.Dfa.dialect("csv")                # (kept alive across the call)
        rc = L.parpa_parse(dfa_csv.handle, ctypes.byref(sch), ctypes.c_void_p(d.data_ptr()), d.numel(), None,
                           ctypes.byref(r))
        assert rc == parpa.ENOMEM, rc
    finally:
        assert L.parpa_set_allocator(None, None, None) == 0

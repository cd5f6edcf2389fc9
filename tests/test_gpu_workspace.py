"""GPU: parse_into with a caller-owned workspace (parpa_parse_into_ws) — reused across parses of different
sizes and paths (k_small below 2 MB, the staged kernels above), inside a CUDA graph, bit-exact vs the oracle."""
import numpy as np
import pytest

import datagen
import oracle
from tests.gpu_helpers import compare

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
import paper_1905_13415_b200 as parpa  # noqa: E402


def dev(a):
    t = torch.empty(max(len(a), 1), dtype=torch.uint8, device="cuda")
    if len(a):
        t[:len(a)].copy_(torch.from_numpy(np.frombuffer(bytes(a), np.uint8).copy()))
    return t[:len(a)]


def test_workspace_reuse_across_sizes_and_paths():
    ws = parpa.Workspace(6_000_000)
    for name, n in [("cfg1", 300_000), ("cfg1", 1_000_000), ("yelp", 5_000_000), ("cfg1", 700_000), ("clf", 1_500_000),
                    ("taxi", 4_000_000), ("cfg1", 64), ("cfg1", 0), ("cfg1", 1_900_000)]:
        w = datagen.WORKLOADS[name]
        data, g = datagen.generate(name, n) if n else (np.zeros(0, np.uint8), None)
        ora = oracle.parse(w.dialect, data, w.C, list(w.types))
        schema = parpa.Schema(list(w.types))
        cap = ora.R + 2
        cols = parpa.alloc_columns(schema, cap)
        st = parpa.new_stats_tensor()
        parpa.parse_into(parpa.Dfa.dialect(w.dialect), schema, dev(data), cols, cap, st, workspace=ws)
        compare(parpa.ParseResult(cols, parpa.stats_from_tensor(st)), ora, w.types, f"{name}-{n}")
    with pytest.raises(parpa.ParpaError):                    # longer than the workspace
        data, _ = datagen.generate("cfg1", 7_000_000)
        parpa.parse_into(parpa.Dfa.dialect("csv"), parpa.Schema(list(datagen.WORKLOADS["cfg1"].types)), dev(data),
                         parpa.alloc_columns(parpa.Schema(list(datagen.WORKLOADS["cfg1"].types)), 10),
                         10, parpa.new_stats_tensor(), workspace=ws)
    ws.close()


def test_workspace_cuda_graph_replays():
    w = datagen.WORKLOADS["cfg1"]
    data, g = datagen.generate("cfg1", 1_000_000)
    ora = oracle.parse("csv", data, w.C, list(w.types))
    d = dev(data)
    dfa = parpa.Dfa.dialect("csv")
    schema = parpa.Schema(list(w.types))
    cap = ora.R + 2
    cols = parpa.alloc_columns(schema, cap)
    st = parpa.new_stats_tensor()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        ws = parpa.Workspace(2_000_000, stream=s)
        n = parpa.parse_into(dfa, schema, d, cols, cap, st, stream=s, workspace=ws)
        assert n == 1                                         # one cooperative kernel
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            parpa.parse_into(dfa, schema, d, cols, cap, st, stream=s, workspace=ws)
    for _ in range(5):
        for c in cols:
            c.offset.zero_()
            if c.value is not None:
                c.value.zero_()
        st.zero_()
        graph.replay()
        torch.cuda.synchronize()
        compare(parpa.ParseResult(cols, parpa.stats_from_tensor(st)), ora, w.types, "graph")

"""Parsing rate vs input size (the paper's fig:inputsize: 1-512 MB of yelp and NYC taxi) on
synthetic inputs: device time of one parse_into (all kernels, inputs resident, CUDA events, median of
repeats), eager launches and CUDA-graph replays.
usage: python scripts/size_sweep.py [workload ...]"""
import json
import statistics
import sys

sys.path.insert(0, ".")
import torch

import datagen
import paper_1905_13415_b200 as parpa

SIZES = [1 << 20, 2 << 20, 5 << 20, 10 << 20, 32 << 20, 128 << 20, 512 << 20, 2 << 30]
out = []
for name in (sys.argv[1:] or ["yelp", "taxi"]):
    w = datagen.WORKLOADS[name]
    dfa = parpa.Dfa.dialect(w.dialect)
    schema = parpa.Schema(list(w.types))
    for size in SIZES:
        data, g = datagen.generate(name, size)                # whole records, <= size bytes
        d = torch.from_numpy(data.copy()).cuda()
        n = d.numel()
        res = parpa.parse(dfa, schema, d)
        cap = res.records + 1
        cols = parpa.alloc_columns(schema, cap)
        st = parpa.new_stats_tensor()
        s = torch.cuda.current_stream()
        reps = 20 if n < (256 << 20) else 5
        for _ in range(3):
            parpa.parse_into(dfa, schema, d, cols, cap, st)
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            parpa.parse_into(dfa, schema, d, cols, cap, st)
            e1.record(s)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = statistics.median(ts)
        row = {"workload": name, "bytes": n, "records": res.records, "ms": round(ms, 4), "GB/s": round(n / ms / 1e6, 2)}
        if n <= (32 << 20):                                    # launch-bound sizes: CUDA graph of one parse
            g_ = torch.cuda.CUDAGraph()
            cs = torch.cuda.Stream()
            cs.wait_stream(s)
            with torch.cuda.stream(cs):
                parpa.parse_into(dfa, schema, d, cols, cap, st, stream=cs)
                torch.cuda.synchronize()
                with torch.cuda.graph(g_, stream=cs):
                    parpa.parse_into(dfa, schema, d, cols, cap, st, stream=cs)
            torch.cuda.synchronize()
            for _ in range(3):
                g_.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(100):
                g_.replay()
            e1.record()
            torch.cuda.synchronize()
            gms = e0.elapsed_time(e1) / 100
            row["graph_ms"] = round(gms, 4)
            row["graph_GB/s"] = round(n / gms / 1e6, 2)
        st_ = parpa.stats_from_tensor(st)
        assert st_["status"] == 0 and st_["records"] == res.records, st_
        print(json.dumps(row), flush=True)
        out.append(row)

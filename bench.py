#!/usr/bin/env python
"""Benchmark of the ParPaRaw hot path on B200 (see DESIGN.md §7 Measurement).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config yelp|taxi|clf|cfg1] [--impl ours|reference]

A step = one full parse (all of S1-S8) of one GPU's input, resident in HBM.  With no --config the
main line is the north-star configuration (yelp-shaped quoted CSV, 4.823 GB: "bit-exact parse of
>= 4.8 GB quoted CSV on one B200", BASELINE.json) and the other single-GPU configs of BASELINE.json
(taxi 4.8 GB = configs[1], CLF ~8 GB = configs[3], the 1 MB cfg1 = configs[0]) follow as same-run
sub-records under "configs", each with its own roofline, step fraction, clocks and parity.

For N > 1 (one rank per GPU, NCCL; `--gpus N` without torchrun re-launches itself under
torch.distributed.run) every rank owns one contiguous, deliberately not record-aligned byte range
of one logical file of the config's shape (weak scaling) and the step includes the two summary
allgathers.

`value` = input GB/s of the whole job (all ranks' bytes / max-over-ranks device time), outputs
written column-major into pre-sized device columns (capacity from an untimed plan pass).  Parity:
after the timed steps every output row of every column is compared with the oracle (the sequential
CPU parser, oracle/), run over generator record ranges on the host's cores.  One JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import hashlib
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "on-device parse GB/s of input (1/2/4/8 B200) and fraction of HBM roofline"
CONFIG_LABEL = {
    "yelp": "Yelp-reviews-shaped CSV, 4.823 GB, all fields quoted, long multi-line text with escaped quotes "
            "(BASELINE configs[2] at the paper's size; the north-star >= 4.8 GB quoted-CSV target)",
    "taxi": "NYC-taxi-shaped CSV, 4.8 GB, 18 numeric/datetime columns, unquoted (BASELINE configs[1])",
    "clf": "Common-Log-Format-shaped logs, ~7.5 GB, 9-state DFA, '#' directive lines (BASELINE configs[3])",
    "cfg1": "1 MB RFC-4180 CSV, 8 columns, ~10% quoted fields (BASELINE configs[0])",
    "taxi64": "64 GB taxi-shaped CSV sharded across the GPUs (strong scaling), in-device windows with "
              "summary carry, cross-GPU transition-vector / count allgather and halo (BASELINE configs[4])",
}
RECORDS_PER_RANK = {"taxi": 48_900_000, "yelp": 6_670_000, "clf": 78_000_000, "cfg1": 10_000}
BYTES_CAP = {"taxi": 4_800_000_000, "yelp": 4_823_000_000, "clf": 8_000_000_000, "cfg1": 1_000_000}
TAXI64_RECORDS = 652_000_000          # ~64e9 bytes of taxi-shaped records (98.1 B each), seed 5
TAXI64_WINDOW = int(os.environ.get("PARPA_BENCH_WINDOW", 8_000_000_000))   # bytes per in-device window
SUB_CONFIGS = ["taxi", "clf", "cfg1"]


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def load_traffic(config, nbytes, timestamps=False):
    """DRAM bytes per launch of the dominant kernel: the committed ncu --set full measurement
    (profiles/ncu_traffic.json, bytes per input byte of that config) times this launch's input."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        r = d.get(config + ("+ts" if timestamps else ""))
        return int(r["dram_bytes_per_input_byte"] * nbytes) if r else None
    except Exception:
        return None


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class Clocks:
    """nvidia-smi sampled every 25 ms during the timed region (clocks + throttle reasons)."""

    def __init__(self):
        self.proc = None
        self.path = None

    def start(self, index=0):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={index}",
                 "--query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "25"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            t0 = time.time()                       # nvidia-smi's start-up can exceed 0.2 s on a busy host:
            while time.time() - t0 < 3.0:          # wait for its first sample before the timed region
                time.sleep(0.05)
                if os.path.getsize(self.path) > 0:
                    break
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        t0 = time.time()                           # short timed regions (cfg1: ~10 ms): let the 25 ms sampler
        while time.time() - t0 < 0.5:              # record at least three samples around the region
            try:
                with open(self.path) as f:
                    if sum(1 for _ in f) >= 3:
                        break
            except OSError:
                break
            time.sleep(0.025)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                parts = [x.strip() for x in line.split(",")]
                if len(parts) < 9:
                    continue
                try:
                    sm.append(float(parts[1]))
                    mx = float(parts[2])
                except ValueError:
                    continue
                for n, v in zip(names, parts[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
        except Exception:
            return None
        finally:
            try:
                os.unlink(self.path)
            except OSError:
                pass
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def gen_range(config, rank, world, pin=True, records=0):
    """This rank's byte range of the logical input (host, pinned) + its left context and base."""
    import torch
    import datagen
    w = datagen.WORKLOADS[config]
    rb = records or RECORDS_PER_RANK[config]
    # (--records: scaled from the config's bytes per record, with headroom; never more than needed)
    cap = BYTES_CAP[config] + (1 << 20) if not records else \
        int(BYTES_CAP[config] * records / RECORDS_PER_RANK[config] * 1.25) + (16 << 20)
    cut = lambda g: 0 if g == 0 else 37 + 11 * g              # mid-record cut points
    host = torch.empty(cap + (1 << 20), dtype=torch.uint8, pin_memory=pin)
    g0 = datagen.fill(w, host.data_ptr(), cap, first_record=rank * rb, max_records=rb)
    block_len = g0.nbytes
    # bytes of the next block that belong to this range
    ext = b""
    if rank + 1 < world:
        nxt = b"".join(datagen.record(w, (rank + 1) * rb + i) for i in range(4))
        ext = nxt[:cut(rank + 1)]
    n_ext = len(ext)
    if n_ext:
        host[block_len:block_len + n_ext] = torch.frombuffer(bytearray(ext), dtype=torch.uint8)
    c0 = cut(rank) if world > 1 else 0
    left = host[:c0].clone() if c0 else None
    data_host = host[c0:block_len + n_ext]
    return data_host, left, block_len, c0, g0


TS_COLS = {"taxi": (1, 2), "yelp": (8,), "clf": (3,), "cfg1": (), "taxi64": (1, 2)}
TIMESTAMP = 3


def workload(config, timestamps=False):
    """The workload of a config; with --timestamps its datetime columns are typed TIMESTAMP
    (int64 epoch seconds) instead of spans."""
    import dataclasses
    import datagen
    w = datagen.WORKLOADS[config]
    if not timestamps:
        return w
    t = list(w.types)
    for c in TS_COLS[config]:
        t[c] = TIMESTAMP
    return dataclasses.replace(w, types=tuple(t))


def run_reference(args):
    """--impl reference: the oracle (the sequential CPU parser) on bounded samples of the workload."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import datagen
    import oracle
    config = args.config or "yelp"
    w = workload(config, args.timestamps)
    sample = args.ref_sample_bytes
    data, g = datagen.generate(config, sample)
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        r = oracle.parse(w.dialect, data, w.C, list(w.types))
        dt = time.perf_counter() - t0
        assert r.status == 0 and r.R == g.records
        if i >= args.warmup:
            times.append(dt)
    ms = statistics.mean(times) * 1e3
    v = len(data) / (ms * 1e-3) / 1e9
    line = {"metric": METRIC, "value": round(v, 4), "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic", "impl": "reference",
            "config": {"workload": config, "description": CONFIG_LABEL[config], "timestamps": bool(args.timestamps),
                       "sample_bytes": len(data), "records": g.records},
            "cpu_baseline": {"value": round(v, 4), "unit": "GB/s", "cores": 1, "kind": "oracle",
                             "cpu": cpu_model(),
                             "sample": f"first {len(data)} bytes ({g.records} records) of the {config} workload, "
                                       f"single-threaded sequential parse incl. int64/float64 conversion"},
            "e2e": {"value": round(v, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(config, data_host, budget_s=10.0, timestamps=False):
    """The oracle as it stands, 1 host core, on a bounded prefix of this workload."""
    import oracle
    w = workload(config, timestamps)
    arr = data_host.numpy()
    probe = min(arr.size, 20_000_000)
    t0 = time.perf_counter()
    oracle.parse(w.dialect, arr[:probe], w.C, list(w.types))
    rate = probe / max(time.perf_counter() - t0, 1e-6)
    n = int(min(arr.size, max(probe, rate * budget_s)))
    t0 = time.perf_counter()
    r = oracle.parse(w.dialect, arr[:n], w.C, list(w.types))
    dt = time.perf_counter() - t0
    return {"value": round(n / dt / 1e9, 4), "unit": "GB/s", "cores": 1, "kind": "oracle", "cpu": cpu_model(),
            "sample": f"first {n} bytes ({r.R} records) of this rank's input; single-threaded sequential "
                      f"parse with int64/float64 conversion; oracle uses 1 of {os.cpu_count()} host cores"}


# ---- same-run parity: every output row against the oracle, over generator record ranges -----------------
def _digest(a):
    return hashlib.blake2b(memoryview(a).cast("B"), digest_size=16).hexdigest()


def _oracle_chunk(config, w, r0, m):
    """Worker: the generator's records [r0, r0 + m) parsed by the oracle; per-column digests with
    offsets relative to the chunk's first byte (the chunk starts a record, so the state is the start)."""
    import numpy as np
    import datagen
    import oracle
    cap = int(BYTES_CAP[config] / RECORDS_PER_RANK[config] * m * 1.5) + (4 << 20)
    while True:
        data, g = datagen.generate(config, cap, first_record=r0, threads=1, max_records=m)
        if g.records == m:
            break
        cap *= 2                                             # a chunk of long records: retry larger
    r = oracle.parse(w.dialect, data, w.C, list(w.types))
    cols = []
    for c in range(w.C):
        d = [_digest(r.offset[c]), _digest(r.length[c])]
        if r.value[c] is not None:
            d += [_digest(r.value[c]), _digest(r.valid[c])]
        cols.append(d)
    return len(data), r.R, r.status, r.n_missing, r.n_extra, cols


def full_parity(config, w, cols, stats, R, workers=None):
    """Compare every row of every device column with the oracle, chunk by chunk in parallel threads (the
    oracle and the generator release the GIL).  Returns a dict for the JSON line."""
    import numpy as np
    t0 = time.perf_counter()
    workers = workers or max(1, (os.cpu_count() or 2) - 1)
    m = max(1000, -(-R // (workers * 6)))
    starts = list(range(0, R, m))
    with cf.ThreadPoolExecutor(workers) as ex:
        res = list(ex.map(lambda r0: _oracle_chunk(config, w, r0, min(m, R - r0)), starts))
    base = np.cumsum([0] + [x[0] for x in res[:-1]]).astype(np.uint64)
    bad = []
    if sum(x[1] for x in res) != R:
        bad.append(f"records oracle {sum(x[1] for x in res)} vs device {R}")
    if any(x[2] != 0 for x in res) or sum(x[3] for x in res) != stats["missing_records"] \
            or sum(x[4] for x in res) != stats["extra_fields"]:
        bad.append("status / missing / extra counts")
    for c in range(w.C):
        off = cols[c].offset.cpu().numpy().view(np.uint64)[:R]
        ln = cols[c].length.cpu().numpy().view(np.uint32)[:R]
        val = cols[c].value.cpu().numpy().view(np.int64)[:R] if cols[c].value is not None else None
        ok = cols[c].valid.cpu().numpy()[:R] if cols[c].valid is not None else None
        for k, r0 in enumerate(starts):
            r1 = min(R, r0 + m)
            d = [_digest(off[r0:r1] - base[k]), _digest(np.ascontiguousarray(ln[r0:r1]))]
            if val is not None:
                d += [_digest(np.ascontiguousarray(val[r0:r1])), _digest(np.ascontiguousarray(ok[r0:r1]))]
            if d != res[k][5][c]:
                bad.append(f"column {c} rows [{r0}, {r1})")
                break
        del off, ln, val, ok
    return {"checked": f"all {R} rows x {w.C} columns (offset, length; value + valid of typed columns) and "
                       f"the record / missing / extra counts vs the oracle, {len(starts)} generator record "
                       f"ranges on {workers} host threads", "mismatches": len(bad), "detail": bad[:5],
            "ok": not bad, "seconds": round(time.perf_counter() - t0, 1)}


def run_e2e(parpa, dfa, schema, data_host, cap, w, steps):
    """End to end through the public API with HOST buffers: pinned input -> H2D -> parse -> D2H of
    every output column into pinned host columns, every step (parpa_parse_host)."""
    import torch
    import datagen
    host_cols = []
    out_bytes = 0
    for t in w.types:
        off = torch.empty(cap, dtype=torch.int64, pin_memory=True)
        ln = torch.empty(cap, dtype=torch.int32, pin_memory=True)
        out_bytes += cap * 12
        if t == datagen.SPAN:
            host_cols.append(parpa.Column(off, ln))
        else:
            val = torch.empty(cap, dtype=torch.float64 if t == datagen.FLOAT64 else torch.int64, pin_memory=True)
            ok = torch.empty(cap, dtype=torch.uint8, pin_memory=True)
            out_bytes += cap * 9
            host_cols.append(parpa.Column(off, ln, val, ok))
    times = []
    warm = 2                                 # the first calls map the pool's partition buffers
    for i in range(steps + warm):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        stats = parpa.parse_host_into(dfa, schema, data_host, host_cols, cap)
        dt = time.perf_counter() - t0
        assert stats["status"] == 0 and stats["records"] == cap, stats
        if i >= warm:
            times.append(dt)
    t = statistics.mean(times)
    return {"value": round(data_host.numel() / t / 1e9, 3), "unit": "GB/s",
            "h2d_bytes_per_step": int(data_host.numel()), "d2h_bytes_per_step": int(out_bytes + 64),
            "ms_per_step": round(t * 1e3, 2), "api": "parpa_parse_host (pinned host input and columns)"}


def run_config(args, config, ctx, main=True):
    """Generate, parse (untimed plan + warm-up), time `steps` parses, check parity; returns the record."""
    import numpy as np
    import torch
    import datagen
    import paper_1905_13415_b200 as parpa
    from paper_1905_13415_b200 import distributed as pdist

    world, rank, dist, coll, gpu = ctx["world"], ctx["rank"], ctx["dist"], ctx["coll"], ctx["gpu"]
    w = workload(config, args.timestamps)
    dfa = parpa.Dfa.dialect(w.dialect)
    schema = parpa.Schema(list(w.types))

    t_gen = time.time()
    data_host, left_host, block_len, cut0, g = gen_range(config, rank, world, records=args.records)
    t_gen = time.time() - t_gen
    n = data_host.numel()
    d = torch.empty(n + 64, dtype=torch.uint8, device="cuda")[:n]
    d.copy_(data_host, non_blocking=True)
    left = left_host.cuda() if left_host is not None else None
    base = 0
    if world > 1:
        lens = torch.tensor([block_len], dtype=torch.int64, device=coll)
        all_lens = [torch.zeros_like(lens) for _ in range(world)]
        dist.all_gather(all_lens, lens)
        base = sum(int(x.item()) for x in all_lens[:rank]) + cut0
    torch.cuda.synchronize()

    # capacity from an untimed scan pass (records of this range)
    stream = torch.cuda.current_stream()
    if world == 1:
        res_plan = parpa.parse(dfa, schema, d)
        cap = res_plan.records
        assert res_plan.status == 0 and cap == g.records, (res_plan.stats, g.records)
        del res_plan
    else:
        cap = g.records + 2
    cols = parpa.alloc_columns(schema, cap)
    st = parpa.new_stats_tensor()
    is_last = rank == world - 1

    def step():
        if world == 1:
            return parpa.parse_into(dfa, schema, d, cols, cap, st)
        pdist.parse_sharded(dfa, schema, d, base, cols, cap, st, left=None, is_last=is_last,
                            exchange_device=coll)          # the halo is exchanged between the ranks
        return 7                                  # range_begin 2 + range_count 2 + range_emit 3

    parpa.set_profiling(False)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    stats = parpa.stats_from_tensor(st)
    assert stats["status"] == 0, stats
    if world == 1:
        assert stats["records"] == g.records, (stats, g.records)
    else:                                                     # the ranks' records add up exactly
        tr = torch.tensor([stats["records"], g.records], dtype=torch.float64, device=coll)
        dist.all_reduce(tr, op=dist.ReduceOp.SUM)
        assert int(tr[0].item()) == int(tr[1].item()), (stats, tr)

    # launch-bound inputs (cfg1, 1 MB): each step is one replay of a CUDA graph of the parse
    use_graph = world == 1 and (args.graph or (config == "cfg1" and not args.no_graph))
    graph, per_step = None, 0
    if use_graph:
        gs = torch.cuda.Stream()
        gs.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        # a caller-owned workspace (parpa_parse_into_ws): the graph is the parse kernel(s) alone, no
        # allocation / memset nodes
        ws = parpa.Workspace(d.numel(), stream=gs)
        with torch.cuda.stream(gs):
            parpa.parse_into(dfa, schema, d, cols, cap, st, stream=gs, workspace=ws)
            torch.cuda.synchronize()
            with torch.cuda.graph(graph, stream=gs):
                per_step = parpa.parse_into(dfa, schema, d, cols, cap, st, stream=gs, workspace=ws)
        torch.cuda.synchronize()
        for _ in range(args.warmup):
            graph.replay()
        torch.cuda.synchronize()
        assert parpa.stats_from_tensor(st)["records"] == g.records

    # the timed region: production launch sequence, no profiling events between the kernels
    steps = args.steps * (20 if use_graph else 1)
    clocks = Clocks()
    clocks.start(gpu)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    e0.record(stream)
    for _ in range(steps):
        if use_graph:
            graph.replay()
            launches += per_step
        else:
            launches += step()
    e1.record(stream)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms_total = e0.elapsed_time(e1)
    clk = clocks.stop()
    # per-kernel device times from separate profiled steps (CUDA events around every launch)
    parpa.set_profiling(True)
    for _ in range(2 if config != "cfg1" else 5):
        step()
    torch.cuda.synchronize()
    ktimes = parpa.last_kernel_times()
    parpa.set_profiling(False)
    ms_step = ms_total / steps
    if dist:
        t = torch.tensor([ms_step], dtype=torch.float64, device=coll)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
        tb = torch.tensor([n], dtype=torch.float64, device=coll)
        dist.all_reduce(tb, op=dist.ReduceOp.SUM)
        total_bytes = float(tb.item())
    else:
        total_bytes = float(n)
    value = total_bytes / (ms_step * 1e-3) / 1e9

    # roofline of the dominant kernel (algorithmic bytes)
    stats = parpa.stats_from_tensor(st)
    T = sum(1 for t in w.types if t != datagen.SPAN)
    R = stats["records"]
    alg_bytes = n + R * w.C * 12 + R * T * 9
    per_kernel = {}
    for name, ms in ktimes:
        per_kernel.setdefault(name, []).append(ms)
    # the emission kernel: it reads the input and writes every output column — k_emit (2 KB
    # warp tiles) or k_emit_sparse (8 KB super tiles, >= 32 bytes per field); the other returns at once
    dom = max(("k_emit", "k_emit_sparse"), key=lambda k: statistics.mean(per_kernel[k]) if per_kernel.get(k) else -1.0)
    kt = per_kernel.get(dom, [])
    peak, peak_src = load_peaks()
    roof = None
    if kt:
        kms = statistics.mean(kt)
        achieved = alg_bytes / (kms * 1e-3) / 1e9
        tr = load_traffic(config, n, args.timestamps)
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": tr, "kernel": dom, "kernel_ms": round(kms, 4),
                "algorithmic_bytes_per_launch": int(alg_bytes), "peak_source": peak_src,
                "share_of_step": round(kms / ms_step, 4),
                "step_achieved": round(alg_bytes * (total_bytes / n) / (ms_step * 1e-3) / 1e9, 1),
                "step_frac": round(alg_bytes * (total_bytes / n) / (ms_step * 1e-3) / 1e9 / peak, 4)}
        # every kernel's share of the step and its own algorithmic fraction: the passes each read the input once
        # (N bytes; their masks / transition vectors are intermediates), the emission kernel moves bytes_alg
        kk = {}
        for name, v in per_kernel.items():
            m = statistics.mean(v)
            ab = alg_bytes if name in ("k_emit", "k_emit_sparse") else (n if name in ("k_pass1", "k_pass2") else None)
            kk[name] = {"ms": round(m, 4), "share": round(m / ms_step, 4)}
            if ab is not None and m > 0.05:
                kk[name].update({"alg_bytes": int(ab), "frac": round(ab / (m * 1e-3) / 1e9 / peak, 4)})
        roof["kernels"] = kk
        roof["largest_share"] = max(kk, key=lambda k: kk[k]["share"])

    parity = None
    if world == 1 and args.parity == "full":
        parity = full_parity(config, w, cols, stats, R)
        if not parity["ok"]:
            print(f"PARITY FAILURE {config}: {parity['detail']}", file=sys.stderr, flush=True)

    cpu = None
    if rank == 0 and not args.no_cpu and main:
        cpu = cpu_baseline(config, data_host, timestamps=args.timestamps)
    e2e = None
    if rank == 0 and world == 1 and not args.no_e2e and main:
        e2e = run_e2e(parpa, dfa, schema, data_host, cap, w, args.e2e_steps)

    rec = {"metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": steps,
           "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
           "config": {"workload": config, "description": CONFIG_LABEL[config], "timestamps": bool(args.timestamps),
                      "bytes_per_gpu": n, "records_per_gpu": R, "columns": w.C, "typed_columns": T,
                      "dialect": w.dialect,
                      "path": ("parse_into (" + ", ".join(per_kernel) + ")") if world == 1 else
                              "range_begin + allgather(tau) + range_count + allgather(counts) + range_emit",
                      "l2": "input >> 126 MB L2 (no flush needed)" if n > (512 << 20) else
                            "input < L2: outputs and inputs stay L2-resident between steps (latency-bound size)",
                      "launch": "CUDA graph replay per step (parse_into with a caller workspace)" if use_graph else "eager",
                      "generate_s": round(t_gen, 1),
                      "kernel_ms": {k: round(statistics.mean(v), 4) for k, v in per_kernel.items()},
                      "kernel_ms_source": "separate profiled steps after the timed region"},
           "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clk,
           "parity": parity}
    del cols, d, data_host, left, st
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return rec


def run_taxi64(args, ctx):
    """configs[4]: 64 GB of taxi-shaped CSV, strong scaling.  Rank g of N holds records [g R/N, (g+1) R/N)
    of one logical file, cut mid-record between ranks (the cut bytes belong to the rank after).  Each
    rank's range is parsed in in-device windows of TAXI64_WINDOW bytes with the summary carry (range
    plans: every window's pass 1 -> its transition vector; composed -> the rank's vector -> allgather
    across ranks -> entry state; every window counted from its entry -> the rank's counts -> allgather ->
    prefix; every window emitted into the same column buffers, the bytes before it on the GPU as its left
    context, the cross-rank halo for the first).  One step = the whole 64 GB."""
    import numpy as np
    import torch
    import datagen
    import paper_1905_13415_b200 as parpa
    from paper_1905_13415_b200 import distributed as pdist
    world, rank, dist, coll, gpu = ctx["world"], ctx["rank"], ctx["dist"], ctx["coll"], ctx["gpu"]
    w = datagen.WORKLOADS["taxi64"]
    dfa = parpa.Dfa.dialect(w.dialect)
    schema = parpa.Schema(list(w.types))
    R_all = args.records or TAXI64_RECORDS
    r0, r1 = rank * R_all // world, (rank + 1) * R_all // world
    per_rec = 98.2
    cap = int((r1 - r0) * per_rec * 1.08) + (64 << 20)
    t_gen = time.time()
    host = torch.empty(cap, dtype=torch.uint8, pin_memory=True)
    g = datagen.fill(w, host.data_ptr(), cap, first_record=r0, max_records=r1 - r0)
    assert g.records == r1 - r0, (g.records, r1 - r0)
    cut = lambda k: 0 if k == 0 else 37 + 11 * k
    ext = b""
    if rank + 1 < world:
        ext = b"".join(datagen.record(w, r1 + i) for i in range(4))[:cut(rank + 1)]
    if ext:
        host[g.nbytes:g.nbytes + len(ext)] = torch.frombuffer(bytearray(ext), dtype=torch.uint8)
    c0 = cut(rank) if world > 1 else 0
    n = g.nbytes + len(ext) - c0
    d = torch.empty(n + 64, dtype=torch.uint8, device="cuda")[:n]
    d.copy_(host[c0:c0 + n], non_blocking=True)
    torch.cuda.synchronize()
    del host
    t_gen = time.time() - t_gen
    base = 0
    if world > 1:
        blk = torch.tensor([g.nbytes], dtype=torch.int64, device=coll)
        all_blk = [torch.zeros_like(blk) for _ in range(world)]
        dist.all_gather(all_blk, blk)
        base = sum(int(x.item()) for x in all_blk[:rank]) + c0
    wins = [(lo, min(n, lo + TAXI64_WINDOW)) for lo in range(0, n, TAXI64_WINDOW)] or [(0, 0)]
    cap_w = int(min(TAXI64_WINDOW, n) / 80) + 1024         # rows per window (taxi records are >= 80 bytes)
    HALO_W = 1 << 20                                      # left context of windows after the first
    cols = parpa.alloc_columns(schema, cap_w)
    sts = [parpa.new_stats_tensor() for _ in wins]
    dev = coll

    def step(check=None):
        plans = [parpa.RangePlan(dfa, d[lo:hi], base + lo) for lo, hi in wins]
        try:
            tau = list(range(dfa.num_states))
            for p in plans:
                tau = parpa.compose_tau(dfa, tau, p.tau)
            if world > 1:
                taus = [pdist.tau_from_bytes(b, dfa.num_states)
                        for b in pdist._allgather_bytes(pdist.tau_to_bytes(tau), None, dev)]
                e = pdist.entry_state(dfa, taus, rank)
            else:
                e = dfa.start
            counts, ew = [], e
            for p in plans:
                counts.append(p.count(ew))
                ew = p.tau[ew]
            mine = pdist.prefix_counts(counts, len(counts))
            if world > 1:
                allc = [parpa._lib.Counts_t.from_buffer_copy(b)
                        for b in pdist._allgather_bytes(bytes(mine), None, dev)]
                prefix = pdist.prefix_counts(allc, rank)
                import struct
                bl = [struct.unpack("<QQ", b) for b in pdist._allgather_bytes(struct.pack("<QQ", base, n), None, dev)]
                bases, lens_ = [x[0] for x in bl], [x[1] for x in bl]
                of = [pdist.prefix_counts(allc, k).open_first for k in range(world)]
                halo, hstate = pdist.halo_exchange(_HaloSrc(plans, wins, base), d, rank, bases,
                                                   pdist.halo_plan(bases, lens_, of), None, dev)
            else:
                prefix, halo, hstate = parpa.identity_counts(), None, None
            pw = prefix
            for k, (p, (lo, hi)) in enumerate(zip(plans, wins)):
                if k == 0:
                    left, ls = halo, hstate
                else:                                      # the 1 MB before the window, with its state
                    left, ls = d[lo - HALO_W:lo], plans[k - 1].state_at(base + lo - HALO_W)
                p.emit(schema, pw, cols, cap_w, sts[k], left=left, left_state=ls,
                       is_last=(rank == world - 1 and k == len(wins) - 1))
                if check is not None:
                    check(k, sts[k], pw, parpa.compose_counts(pw, counts[k]))
                pw = parpa.compose_counts(pw, counts[k])
        finally:
            for p in plans:
                p.close()
        return 7 * len(wins)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # verification (untimed): records and the int64 columns' sums / null counts against the generator
    # (G1), summed over all ranks and windows.
    T_int = [c for c, t in enumerate(w.types) if t == datagen.INT64]
    acc = torch.zeros(2 + 2 * len(T_int), dtype=torch.int64, device="cuda")       # records, status, sums, nulls
    last_w = len(wins) - 1

    def check(k, st_t, pw, after):
        s_ = parpa.stats_from_tensor(st_t)
        acc[1] += int(s_["status"] != 0)
        R = s_["records"]
        acc[0] += R
        for i, c in enumerate(T_int):
            # a record straddling a window (or rank) boundary: its columns < pw.column sit one row past the
            # previous window's count, the rest in this window's row 0
            lo_row = 1 if c < pw.column else 0
            hi_row = R + (1 if (not (k == last_w and rank == world - 1) and c < after.column) else 0)
            if hi_row <= lo_row:
                continue
            v = cols[c].value[lo_row:hi_row]
            ok = cols[c].valid[lo_row:hi_row].bool()
            acc[2 + i] += torch.where(ok, v, torch.zeros_like(v)).sum()
            acc[2 + len(T_int) + i] += (~ok).sum()
    step(check)
    truth = torch.tensor([g.records, 0] + [((x + (1 << 63)) % (1 << 64)) - (1 << 63) for x in g.int_sums]
                         + list(g.int_nulls), dtype=torch.int64, device="cuda")
    if dist:
        a2, t2 = acc.to(coll), truth.to(coll)
        dist.all_reduce(a2)
        dist.all_reduce(t2)
        acc, truth = a2, t2
    ok_all = bool(torch.equal(acc.cpu(), truth.cpu()))
    if not ok_all:
        print("taxi64 ground truth mismatch: got", acc.tolist(), "expected", truth.tolist(), file=sys.stderr)
    gt = {"records": int(acc[0].item()), "exp_records": int(truth[0].item()), "windows_failed": int(acc[1].item()),
          "int_sums_and_nulls_equal": bool(torch.equal(acc[2:].cpu(), truth[2:].cpu()))}
    clocks = Clocks()
    clocks.start(gpu)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    launches = 0
    for _ in range(args.steps):
        launches += step()
    e1.record()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps
    tot = float(n)
    if dist:
        t = torch.tensor([ms], dtype=torch.float64, device=coll)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        tb = torch.tensor([tot], dtype=torch.float64, device=coll)
        dist.all_reduce(tb, op=dist.ReduceOp.SUM)
        tot = float(tb[0].item())
    value = tot / (ms * 1e-3) / 1e9
    R_total = R_all
    alg = tot + R_total * w.C * 12 + R_total * sum(1 for t in w.types if t != datagen.SPAN) * 9
    peak, peak_src = load_peaks()
    return {"metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": "taxi64", "description": CONFIG_LABEL["taxi64"], "total_bytes": int(tot),
                       "records": R_total, "windows_per_rank": len(wins), "window_bytes": TAXI64_WINDOW,
                       "path": "range plans per window: range_begin, compose, (allgather tau), range_count, "
                               "(allgather counts, halo all_to_all), range_emit", "generate_s": round(t_gen, 1),
                       "l2": "input >> 126 MB L2 (no flush needed)"},
            "roofline": {"bound": "hbm", "achieved": round(alg / (ms * 1e-3) / 1e9, 1), "peak": peak * world,
                         "unit": "GB/s", "frac": round(alg / (ms * 1e-3) / 1e9 / (peak * world), 4),
                         "traffic": None, "kernel": "whole step (all windows, all ranks)",
                         "algorithmic_bytes_per_launch": int(alg), "peak_source": peak_src + " x n_gpus"},
            "parity": {"checked": "generator ground truth (G1) over all 64 GB: record count, per-int64-column "
                                  "wrapping sums and null counts, status of every window", "ok": ok_all,
                       **gt},
            "cpu_baseline": None, "e2e": None, "gpu_launches": launches, "clocks": clk}


class _HaloSrc:
    """state_at over a rank's windows (the owner of a halo start may be any window's plan)."""
    def __init__(self, plans, wins, base):
        self.plans, self.wins, self.base = plans, wins, base

    def state_at(self, pos):
        for p, (lo, hi) in zip(self.plans, self.wins):
            if self.base + lo <= pos < self.base + hi:
                return p.state_at(pos)
        raise ValueError(pos)


def relaunch(args):
    """--gpus N > 1 without torchrun: one process per GPU under torch.distributed.run."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=None, choices=list(CONFIG_LABEL),
                    help="one config only (default: yelp main line + taxi / clf / cfg1 sub-records at N=1)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-subs", action="store_true", help="main config only")
    ap.add_argument("--parity", default="full", choices=["full", "none"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--ref-sample-bytes", type=int, default=150_000_000)
    ap.add_argument("--records", type=int, default=0, help="override records per rank (profiling runs)")
    ap.add_argument("--timestamps", action="store_true", help="type the datetime columns as TIMESTAMP (SURVEY N2)")
    ap.add_argument("--graph", action="store_true", help="time CUDA-graph replays of the parse (default for cfg1)")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches even for cfg1")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))

    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    # test switch: every rank on cuda:0 with gloo collectives (validates the sharded path on one GPU;
    # never used for a reported number)
    shared = os.environ.get("PARPA_BENCH_SHARED_GPU") == "1"
    gpu = 0 if shared else local
    coll = "cpu" if shared else "cuda"
    torch.cuda.set_device(gpu)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = {"world": world, "rank": rank, "dist": dist, "coll": coll, "gpu": gpu}
    main_cfg = args.config or "yelp"
    subs = [] if (args.config or world > 1 or args.no_subs or args.records) else SUB_CONFIGS
    line = run_taxi64(args, ctx) if main_cfg == "taxi64" else run_config(args, main_cfg, ctx, main=True)
    if subs:
        line["configs"] = [run_config(args, c, ctx, main=False) for c in subs]
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

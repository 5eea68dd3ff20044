#!/usr/bin/env python
"""Checkpointed GB/s of embedding rows (track + compact + quantize + pack).

Workload (BASELINE.json configs[1], "C2"): Criteo-Kaggle-shaped 26 tables
(the published DLRM cardinalities, 33,762,577 rows) x dim 16 fp32, 8-bit
quantization (naive ranges, the reference's 8-bit default), one checkpoint
every 500 batches of 2048 Zipf(1.05) lookups per table.  One step = one
checkpoint interval:
  K1 mark the interval's 26 x 1,024,000 lookups into the dirty bitmaps,
  K2 capture the interval's dirty ids + fold into the baseline scope,
     (N > 1: NCCL all_gather of the per-table dirty counts),
  K3 gather + quantize + pack the dirty rows into CNR1 records.
Metric = sum of checkpointed fp32 row bytes (dirty rows x 64 B) / device time.
Weak scaling: every rank owns a C2-sized row shard of 26 tables with N x the
rows (rows [rank*card, (rank+1)*card) of each table).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference times the reference's CPU path (the oracle port of
deltasnap's tracker + build_shard_payload, oracle/) on the host cores.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CRITEO_KAGGLE = [1460, 583, 10131227, 2202608, 305, 24, 12517, 633, 3, 93145, 5683, 8351593,
                 3194, 27, 14992, 5461306, 10, 5652, 2173, 4, 7046547, 18, 15, 286181, 105, 142572]
# MLPerf DLRM Criteo-Terabyte cardinalities (capped at 40M rows), 187.8M rows
CRITEO_TB = [39884406, 39043, 17289, 7420, 20263, 3, 7120, 1543, 63, 38532951, 2953546, 403346,
             10, 2208, 11938, 155, 4, 976, 14, 39979771, 25641295, 39664984, 585935, 12972, 108, 36]
BATCHES = 500
BATCH = 2048
ZIPF_S = 1.05

# BASELINE.json configs as single-GPU workloads (per-rank shards; weak scaling)
WORKLOADS = {
    # configs[0]: the reference's own CPU-runnable case (8 x 1M x 64, 1000
    # batches of 2048 Zipf lookups per table, incremental, 4-bit uniform
    # asymmetric = naive min/max ranges)
    "C1": dict(desc="C1: synthetic DLRM-style 8 tables x 1M rows x dim 64 fp32, Zipf lookups, 1000 "
                    "batches of 2048, incremental 4-bit uniform asymmetric (naive ranges)",
               cards=[1_000_000] * 8, dim=64, bitwidth=4, adaptive=False, lookups="zipf",
               n_per_table=1000 * BATCH),
    # configs[1]: the metric's headline config (the default)
    "C2": dict(desc="C2: Criteo-Kaggle-shaped 26 tables x dim 16 fp32, 8-bit naive, checkpoint "
                    "every 500 batches x 2048 Zipf(1.05) lookups/table",
               cards=CRITEO_KAGGLE, dim=16, bitwidth=8, adaptive=False, lookups="zipf",
               n_per_table=BATCHES * BATCH),
    # the north-star target T, one GPU's shard of 1B x 128 over 8 GPUs:
    # 125M rows, 4-bit incremental, ~26% of rows dirty per interval
    "T": dict(desc="T (one of 8 GPU shards): 125M rows x dim 128 fp32 (64 GB), 4-bit naive "
                   "incremental, 37.5M uniform lookups per interval (26% of rows dirty)",
              cards=[125_000_000], dim=128, bitwidth=4, adaptive=False, lookups="uniform",
              n_per_table=37_500_000),
    "T-adaptive": dict(desc="T shard with the reference's 4-bit default ranges: adaptive greedy "
                            "(bins 45, ratio 0.2)",
                       cards=[125_000_000], dim=128, bitwidth=4, adaptive=True, lookups="uniform",
                       n_per_table=37_500_000),
    # configs[3], one of 8 GPU shards of 1B x 128: the 2-bit adaptive greedy
    # ranges (bins 25, ratio 0.5: 25 candidate evaluations per row)
    "C4": dict(desc="C4 (one of 8 GPU shards): 125M rows x dim 128 fp32 (64 GB), 2-bit adaptive "
                    "greedy (bins 25, ratio 0.5) incremental, 37.5M uniform lookups per interval",
               cards=[125_000_000], dim=128, bitwidth=2, adaptive=True, lookups="uniform",
               n_per_table=37_500_000),
    # configs[4]: restore of a full checkpoint + 5 incremental deltas
    "C5": dict(desc="C5: restore a chain (1 full + 5 incremental 8-bit checkpoints of the C2 "
                    "tables) into device tables: unpack, dequantize, scatter, baseline bits",
               cards=CRITEO_KAGGLE, dim=16, bitwidth=8, adaptive=False, lookups="zipf",
               n_per_table=BATCHES * BATCH, restore=5),
    # configs[2], one of 8 GPU shards: Criteo-TB rows / 8, 4-bit adaptive greedy
    "C3": dict(desc="C3 (one of 8 GPU shards): Criteo-TB-shaped 26 tables / 8 x dim 128 fp32, "
                    "4-bit adaptive greedy (bins 45, ratio 0.2), 500 x 2048 Zipf lookups/table",
               cards=[max(1, c // 8) for c in CRITEO_TB], dim=128, bitwidth=4, adaptive=True,
               lookups="zipf", n_per_table=BATCHES * BATCH),
}
METRIC = "checkpointed GB/s of embedding rows (track+quantize+pack) at 1/2/4/8 B200 vs CPU ref"


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=("ours", "reference"), default="ours")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--tables", type=int, default=0,
                   help="use the first T tables (smoke/profiling only)")
    p.add_argument("--workload", choices=sorted(WORKLOADS), default="C2",
                   help="BASELINE.json config (C2 is the metric's headline config)")
    p.add_argument("--l2-fetch", type=int, default=0,
                   help="cudaLimitMaxL2FetchGranularity in bytes (0 = leave the default; r01's 64 "
                        "changed no DRAM traffic, see roofline.traffic_vs_algorithmic)")
    p.add_argument("--verify-rows", type=int, default=1_000_000,
                   help="records of the last timed step's payload re-derived by the CPU oracle "
                        "(plus every header, the whole dirty-id column, section ends and the "
                        "records around byte 2^31 / 2^32); 0 = no parity check")
    p.add_argument("--no-shipped", action="store_true",
                   help="skip timing the reference package as shipped (baseline/_ref)")
    return p.parse_args()


def workload_of(args):
    w = dict(WORKLOADS[args.workload])
    if args.tables:
        w["cards"] = w["cards"][:args.tables]
    return w


def workload_desc(w):
    return {
        "workload": w["desc"], "name": [k for k, v in WORKLOADS.items() if v["desc"] == w["desc"]][0],
        "tables": len(w["cards"]), "rows_per_rank": int(sum(w["cards"])), "dim": w["dim"],
        "bitwidth": w["bitwidth"], "ranges": "adaptive greedy" if w["adaptive"] else "naive min/max",
        "lookups": w["lookups"], "lookups_per_step_per_rank": int(w["n_per_table"] * len(w["cards"])),
        "lookup_dtype": "per table: ids bit-packed at ceil(log2(rows)) bits (LookupStream)",
        "scope": "interval (consecutive increments)",
        "row_map": "Zipf rank -> row through a seeded permutation per table"
                   if w["lookups"] == "zipf" else "uniform row ids",
        "l2": "flushed between timed steps (256 MB write; L2 126 MB); tables and the packed "
              "lookup stream are both larger than L2",
        "timing": "CUDA events at each step's bounds (K1 -> K2 -> K3 launched back to back, "
                  "programmatic dependent launch); `phases` from a second pass of K steps with "
                  "events between the kernels",
    }


# --------------------------------------------------------------------------------
# clocks (NVML polled every ~1 ms during the timed region)
# --------------------------------------------------------------------------------

class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # NVML unavailable: report what we have
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.001)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.nv is not None:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# --------------------------------------------------------------------------------
# synthetic workload
# --------------------------------------------------------------------------------

def lookups_torch(kind, rows, n, gen, device):
    import torch
    if kind == "uniform":
        return torch.randint(0, rows, (n,), generator=gen, device=device, dtype=torch.int32)
    w = torch.arange(1, rows + 1, dtype=torch.float64, device=device).pow_(-ZIPF_S)
    cdf = torch.cumsum(w, 0)
    cdf /= cdf[-1].clone()
    u = torch.rand(n, dtype=torch.float64, generator=gen, device=device)
    ranks = torch.searchsorted(cdf, u, right=True).clamp_(max=rows - 1)
    perm = torch.randperm(rows, generator=gen, device=device)
    return perm[ranks].to(torch.int32)


HOST_INPUT_BYTES = 8 << 30  # tables up to this size are drawn on the host (numpy)


def table_bytes(w) -> int:
    return int(sum(w["cards"])) * w["dim"] * 4


def host_inputs(w, seed, rank=0):
    """Tables U[-1, 1) (model.py:127-128) and the interval's lookups drawn with
    numpy from (seed, rank): both arms of the bench (ours, --impl reference)
    see the same bytes for the same rank."""
    rng = np.random.default_rng([seed, rank])
    tables = [(rng.random((r, w["dim"]), dtype=np.float32) * 2 - 1) for r in w["cards"]]
    lookups = [lookups_numpy(w["lookups"], r, w["n_per_table"], rng) for r in w["cards"]]
    return tables, lookups


def lookups_numpy(kind, rows, n, rng):
    if kind == "uniform":
        return rng.integers(0, rows, n).astype(np.int32)
    w = np.arange(1, rows + 1, dtype=np.float64) ** -ZIPF_S
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    ranks = np.minimum(np.searchsorted(cdf, rng.random(n), side="right"), rows - 1)
    return rng.permutation(rows)[ranks].astype(np.int32)


# --------------------------------------------------------------------------------
# CPU path (the oracle port of the reference: tracker.py + build_shard_payload)
# --------------------------------------------------------------------------------

class CpuPath:
    """Reference CPU path on host arrays, all host threads.

    Per step: DirtyBitmap.mark of every table's lookups (tracker.py:27-36),
    capture of the interval scope (tracker.py:54-58) + reset_interval
    (:120-124), then build_shard_payload's incremental section per table
    (engine.py:139-187).  Tables run in parallel threads (ctypes releases the
    GIL); rows of a section run on OpenMP threads.

    tables: host arrays, or None with fetch(t, ids) for tables too large to
    copy to the host (the T / C4 shards hold 64 GB): the sampled dirty rows
    are then gathered before the timed build, which codes them in place.
    """

    def __init__(self, tables, lookups, cards, threads, bitwidth=8, adaptive=None, fetch=None):
        from oracle import oracle as O
        self.bitwidth, self.adaptive = bitwidth, adaptive
        self.O = O
        self.tables, self.lookups, self.cards = tables, lookups, cards
        self.fetch = fetch
        self.threads = threads
        self.bits = [np.zeros((r + 7) // 8, np.uint8) for r in cards]
        self.base = [np.zeros((r + 7) // 8, np.uint8) for r in cards]
        from concurrent.futures import ThreadPoolExecutor
        self.pool = ThreadPoolExecutor(max_workers=threads)

    def step(self, tables_subset=None, max_build_rows=None):
        """One interval: returns (dirty rows, payload bytes built, seconds).

        With max_build_rows the sections are built for an evenly strided
        sample of the dirty rows and the build time is scaled to all of them
        (rows are independent in the reference codec, quant.py:14-15)."""
        O = self.O
        ts = range(len(self.cards)) if tables_subset is None else tables_subset
        t0 = time.perf_counter()

        def track(t):
            O.mark(self.bits[t], self.cards[t], self.lookups[t])
            ids = O.dirty_rows(self.bits[t], self.cards[t])
            self.base[t] |= self.bits[t]
            self.bits[t][:] = 0
            return ids

        ids_all = list(self.pool.map(track, ts))
        t1 = time.perf_counter()
        rows = sum(i.size for i in ids_all)
        scale = 1.0
        ids = ids_all
        if max_build_rows and rows > max_build_rows:
            stride = int(np.ceil(rows / max_build_rows))
            ids = [i[::stride] for i in ids_all]
            scale = rows / max(1, sum(i.size for i in ids))
        vals = None
        if self.tables is None:  # untimed gather of the sampled rows from the device
            vals = [self.fetch(t, ids[k]) for k, t in enumerate(ts)]
        big = [k for k, t in enumerate(ts) if ids[k].size > 65536]
        small = [k for k, t in enumerate(ts) if ids[k].size <= 65536]

        def build(k, nthreads):
            t = list(ts)[k]
            if vals is not None:
                return O.build_section(t, vals[k], None, bitwidth=self.bitwidth,
                                       adaptive=self.adaptive, nthreads=nthreads)
            return O.build_section(t, self.tables[t], ids[k], bitwidth=self.bitwidth,
                                   adaptive=self.adaptive, nthreads=nthreads)

        t2 = time.perf_counter()
        outs = list(self.pool.map(lambda k: build(k, 1), small))
        for k in big:
            outs.append(build(k, self.threads))
        t3 = time.perf_counter()
        return rows, sum(len(o[0]) for o in outs), (t1 - t0) + (t3 - t2) * scale


def import_shipped_reference():
    """The unmodified reference package from its offline install
    (baseline/_ref, `pip install --no-index ... --target baseline/_ref`), or
    None when it is not installed."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "deltasnap")):
        return None
    sys.dont_write_bytecode = True
    if path not in sys.path:
        sys.path.append(path)
    try:
        import deltasnap
    except Exception:
        return None
    return deltasnap


def shipped_measure(w, tables, lookups, payload=None, sample_rows=None, fetch=None):
    """The reference as shipped: deltasnap's own
    DirtyBitmap.mark + dirty_rows (tracker.py:27-58) over the interval's
    lookups, then its build_shard_payload (engine.py:118-189) -- one shard,
    so one writer thread (RunConfig.workers = shards, engine.py:231-233) --
    over an evenly strided sample of the dirty rows, the build time scaled to
    all of them (bytes are per-row, quant.py:14-15).  With `payload` (this
    step's device-written payload, N = 1) the sampled records are compared
    byte for byte with the reference's own.  tables=None: the sampled rows
    are gathered from the device (fetch) before the timed build."""
    ds_ref = import_shipped_reference()
    if ds_ref is None:
        return None
    from types import SimpleNamespace
    sample_rows = sample_rows or (20_000 if w["adaptive"] else 100_000)
    t0 = time.perf_counter()
    ids = []
    for t, (r, lk) in enumerate(zip(w["cards"], lookups)):
        bm = ds_ref.tracker.DirtyBitmap(t, r)
        bm.mark(lk)
        ids.append(bm.dirty_rows()[0])
    t_track = time.perf_counter() - t0
    total = sum(i.size for i in ids)
    stride = max(1, int(np.ceil(total / sample_rows)))
    sel = [i[::stride] for i in ids]
    n_sel = sum(x.size for x in sel)
    if tables is None:  # the sampled rows only, as a table of their own
        tabs = [fetch(t, sel[t]) for t in range(len(sel))]
        rows = {t: np.arange(sel[t].size, dtype=np.int64) for t in range(len(sel))}
    else:
        tabs, rows = tables, dict(enumerate(sel))
    snap = SimpleNamespace(shard_tables=lambda sid: [
        ds_ref.model.EmbeddingTable(t, v) for t, v in enumerate(tabs)])
    plan = ds_ref.policy.CheckpointPlan(kind="incremental", rows=rows, bitwidth=w["bitwidth"])
    overrides = None if w["adaptive"] else {w["bitwidth"]: None}
    t1 = time.perf_counter()
    blob, _, _ = ds_ref.engine.build_shard_payload(snap, plan, 0, 1024, overrides)
    t_build = (time.perf_counter() - t1) * total / max(1, n_sel)
    secs = t_track + t_build
    out = {"value": total * w["dim"] * 4 / secs / 1e9, "unit": "GB/s", "cores": 1,
           "kind": "reference", "rows_per_s": total / secs,
           "sample": f"deltasnap (baseline/_ref) as shipped, one writer thread: mark + dirty_rows "
                     f"of all {sum(len(l) for l in lookups)} lookups ({t_track:.2f} s), "
                     f"build_shard_payload of every {stride}-th dirty row ({n_sel} rows, "
                     f"{time.perf_counter() - t1:.2f} s, scaled to {total})"}
    if payload is not None:
        # the reference's records vs the same records of our payload (ids
        # excluded when the sampled rows were re-based into their own table)
        rec = 16 + (w["dim"] * w["bitwidth"] + 7) // 8
        skip = 8 if tables is None else 0
        ref_b = np.frombuffer(blob, np.uint8)
        off_r, off_p, bad, n = 0, 0, 0, 0
        for i in ids:
            pos = np.arange(0, i.size, stride)
            ours = payload[off_p + 24: off_p + 24 + i.size * rec].reshape(i.size, rec)[pos, skip:]
            theirs = ref_b[off_r + 24: off_r + 24 + pos.size * rec].reshape(pos.size, rec)[:, skip:]
            bad += int(np.any(ours != theirs, axis=1).sum())
            n += pos.size
            off_p += 24 + i.size * rec
            off_r += 24 + pos.size * rec
        out["parity_vs_shipped"] = {"records_compared": n, "mismatches": bad,
                                    "ids_compared": skip == 0}
    return out


def cpu_measure(w, tables, lookups, budget_s=20.0, steps=None, shipped=False, payload=None,
                fetch=None):
    """The reference CPU path (oracle port) on all host threads: GB/s of
    checkpointed rows over whole intervals (C2) or, for the large workloads,
    intervals whose section build is sampled to ~budget_s."""
    threads = os.cpu_count() or 1
    acfg = {2: (25, 0.5), 3: (25, 0.2), 4: (45, 0.2)}.get(w["bitwidth"]) if w["adaptive"] else None
    cp = CpuPath(tables, lookups, w["cards"], threads, w["bitwidth"], acfg, fetch=fetch)
    big = sum(w["cards"]) > 50_000_000 or w["adaptive"]
    cap = (200_000 if w["adaptive"] else 2_000_000) if big else None
    cp.step(max_build_rows=cap)  # warm-up (page-in, OpenMP pool)
    rows_c, secs, reps = 0, 0.0, 0
    t0 = time.perf_counter()
    while (steps is None and (reps == 0 or (reps < 3 and time.perf_counter() - t0 < budget_s))) \
            or (steps is not None and reps < steps):
        r, _, dt = cp.step(max_build_rows=cap)
        rows_c += r
        secs += dt
        reps += 1
    sample = (f"{reps} full interval(s): mark {int(sum(len(l) for l in lookups))} lookups, "
              f"capture, {'adaptive' if w['adaptive'] else 'naive'} {w['bitwidth']}-bit sections of "
              + ("every dirty row" if cap is None else f"a strided sample of {cap} dirty rows "
                 "(build time scaled to all dirty rows"
                 + (", the sampled rows gathered from the device table before the build)"
                    if tables is None else ")")))
    out = {"value": rows_c * w["dim"] * 4 / secs / 1e9, "unit": "GB/s", "cores": threads,
           "kind": "port", "sample": sample, "seconds": secs, "steps": reps}
    if shipped:
        out["reference_as_shipped"] = shipped_measure(w, tables, lookups, payload, fetch=fetch)
    return out


def pack_lookups(lookups, cards, dev):
    """The interval's lookup stream through the public API: each table's ids
    bit-packed at ceil(log2(rows)) bits (LookupStream.pack, pinned host
    memory), and its device copy."""
    from paper_2010_08679_b200.tracker import LookupStream
    host = LookupStream.pack({t: lk.cpu().numpy() for t, lk in enumerate(lookups)},
                             dict(enumerate(cards)), pin=True)
    return host, host.to(dev, non_blocking=False)


# --------------------------------------------------------------------------------

def run_reference(args):
    """--impl reference: the CPU path on the host cores, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    w = workload_of(args)
    if table_bytes(w) <= HOST_INPUT_BYTES:
        tables, lookups = host_inputs(w, args.seed, 0)
        fetch, input_gen = None, "numpy default_rng([seed, rank]) (same draw as --impl reference)"
    else:
        # 64 GB shards: only the sampled dirty rows are materialised (random
        # U[-1, 1) rows per request); the lookups are the full interval's
        rng = np.random.default_rng([args.seed, 0])
        lookups = [lookups_numpy(w["lookups"], r, w["n_per_table"], rng) for r in w["cards"]]
        tables = None

        def fetch(t, ids):
            return np.random.default_rng([args.seed, t, len(ids)]).random(
                (len(ids), w["dim"]), dtype=np.float32) * 2 - 1
        input_gen = "torch.Generator on the device"
    dirty = sum(np.unique(lk).size for lk in lookups)
    cpu = cpu_measure(w, tables, lookups, steps=max(1, args.steps), fetch=fetch,
                      shipped=not args.no_shipped)
    value = cpu["value"]
    world = max(1, args.gpus)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s",
        "n_gpus": args.gpus, "steps": cpu["steps"], "warmup": 1,
        "ms_per_step": cpu["seconds"] / cpu["steps"] * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic",
        "config": dict(workload_desc(w), dirty_rows_per_step=dirty * world,
                       parallelism=f"row-sharded x{world}", inputs=input_gen,
                       **({"rank_alignment": "device all_reduce after each untimed L2 flush"}
                          if world > 1 else {})),
        "cpu_baseline": dict({k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")},
                             reference_as_shipped=cpu.get("reference_as_shipped")),
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def step_payload(ck, host_payload, local):
    """This rank's payload of one step as a CNR1 payload: N = 1 writes whole
    sections; N > 1 writes bare record runs, which get headers with the
    rank's own counts here (the assembled shard is the rank-order
    concatenation of such runs, sharded.assemble_shard)."""
    if ck.world == 1:
        return host_payload
    from paper_2010_08679_b200.payload import pack_header
    parts, off = [], 0
    for t, n in zip(ck.tables, local):
        parts.append(np.frombuffer(pack_header(t.table_id, int(n), t.dim, ck.bitwidth,
                                               1 if ck.bitwidth else 0, False), np.uint8))
        parts.append(host_payload[off:off + int(n) * ck.rec])
        off += int(n) * ck.rec
    return np.concatenate(parts)


def verify_step(ck, tables, look_host, w, host_payload, local, sample):
    """Checks one step's payload against the CPU oracle (oracle/verify.py):
    every header, the whole dirty-id column (= np.unique of the interval's
    lookups, tracker.py:54-58), and `sample` strided records plus section
    ends and the records around byte 2^31 / 2^32 re-derived from the same
    table rows (engine.py:118-189)."""
    import torch
    from oracle.verify import verify_payload
    exp = []
    for t, lk in zip(tables, look_host):
        exp.append(dict(table_id=t.table_id, dim=t.dim, ids=np.unique(lk).astype(np.int64) + t.row_base))
    by_id = {t.table_id: t for t in tables}

    def fetch(tid, ids):
        t = by_id[tid]
        idx = torch.from_numpy(np.asarray(ids, np.int64) - t.row_base).to(t.values.device)
        return t.values.index_select(0, idx).cpu().numpy()

    adaptive = None
    if w["adaptive"]:
        adaptive = {2: (25, 0.5), 3: (25, 0.2), 4: (45, 0.2)}[w["bitwidth"]]
    r = verify_payload(step_payload(ck, host_payload, local), exp, bitwidth=w["bitwidth"],
                       adaptive=adaptive, incremental=True, fetch_rows=fetch, sample=sample)
    r["checked_against"] = ("CPU oracle (oracle/deltasnap_oracle.c) re-deriving the records from "
                            "the same table rows; ids against np.unique of the lookups")
    r["rows_checked"] = r["records_checked"]
    return r


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2010_08679_b200 as ds
    from paper_2010_08679_b200.sharded import ShardedCheckpointer
    from paper_2010_08679_b200.tracker import LookupStream

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        # NCCL's banner/debug output goes to stderr: stdout carries only the JSON line
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group("nccl", device_id=dev)
    from paper_2010_08679_b200 import _lib as dslib
    if args.l2_fetch:
        dslib.check(dslib.lib().ds_set_l2_fetch_granularity(args.l2_fetch), "l2 fetch")
    l2_fetch = int(dslib.lib().ds_get_l2_fetch_granularity())

    w = workload_of(args)
    cards, DIM = w["cards"], w["dim"]
    n_look = w["n_per_table"]
    tables = []
    if table_bytes(w) <= HOST_INPUT_BYTES:
        # the same numpy draw as --impl reference (identical inputs per rank)
        h_tables, h_look = host_inputs(w, args.seed, rank)
        for t, (r, v) in enumerate(zip(cards, h_tables)):
            tables.append(ds.DeviceTable(t, torch.from_numpy(v).to(dev), row_base=rank * r,
                                         total_rows=world * r))
        lookups = [torch.from_numpy(lk).to(dev) for lk in h_look]
        del h_tables, h_look
        input_gen = "numpy default_rng([seed, rank]) (same draw as --impl reference)"
    else:
        # 64 GB shards: drawn on the device (Philox)
        gen = torch.Generator(device=dev)
        gen.manual_seed(args.seed * 7919 + rank)
        for t, r in enumerate(cards):
            v = torch.rand((r, DIM), generator=gen, device=dev, dtype=torch.float32).mul_(2).sub_(1)
            tables.append(ds.DeviceTable(t, v, row_base=rank * r, total_rows=world * r))
        lookups = [lookups_torch(w["lookups"], r, n_look, gen, dev) for r in cards]
        input_gen = "torch.Generator on the device"
    # the interval's lookup stream, each table's ids at ceil(log2(rows))
    # bits: ds_mark_packed's input (host copy for e2e, device copy in HBM)
    host_stream, stream = pack_lookups(lookups, cards, dev)
    # ranges: the reference's default for the bitwidth (engine.py:112-115),
    # or naive min/max when the workload says so
    overrides = None if w["adaptive"] else {w["bitwidth"]: None}
    ck = ShardedCheckpointer(tables, w["bitwidth"], adaptive_overrides=overrides, rank=rank,
                             world_size=world, device=dev)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local_rank])

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # warm-up: W steps, then keep stepping until the clocks have ramped
    # (>= 0.3 s).  Every step holds a collective at N > 1, so all ranks run
    # the same number of ramp steps (the max of their own estimates).
    for _ in range(max(3, args.warmup)):
        ck.step(stream)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ck.step(stream)
    torch.cuda.synchronize()
    n_ramp = int(0.3 / max(time.perf_counter() - t0, 1e-6)) + 1
    if world > 1:
        nt_ = torch.tensor([n_ramp], dtype=torch.int64, device=dev)
        dist.all_reduce(nt_, op=dist.ReduceOp.MAX)
        n_ramp = int(nt_.item())
    for _ in range(min(n_ramp, 20000)):
        ck.step(stream)
    torch.cuda.synchronize()
    ck.fetch()  # raises any flagged data error of the warm-up steps

    # ---- device-timed region: exactly K steps --------------------------------------
    # Between timed steps a 256 MB write evicts L2 (126 MB), so no step sees
    # the previous step's lookups, bitmaps or rows; the step time is the sum
    # of the per-step event intervals (the flush itself is not timed).
    K = args.steps
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    align = torch.zeros(1, dtype=torch.int32, device=dev)

    def timed_steps(phased: bool):
        """K steps, each after an untimed L2 flush; events at the step bounds
        (and, phased, between K1 / K2 / K3 -- an event between two kernels
        also stops the second one launching early, so the metric comes from
        the unphased pass)."""
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4 if phased else 2)]
              for _ in range(K)]
        for k in range(K):
            flush.fill_(k & 0xFF)
            if world > 1:
                # ranks leave the (untimed) flush together, as a training
                # step's gradient collective would release them: a device-side
                # all_reduce, no host sync.  Without it one rank's slower flush
                # shows up as another rank's wait inside K3's count exchange.
                dist.all_reduce(align)
            ev[k][0].record()
            ck.mark(stream)                                # K1
            if phased:
                ev[k][1].record()
            ck.counts = ck.tracker.capture_into(ck.ids, None, fold=1, scope=ck.scope)  # K2
            if phased:
                ev[k][2].record()
            ck.write()  # K3 (N > 1: + the count exchange over NVLink peer memory, same launch)
            ev[k][-1].record()
        torch.cuda.synchronize()
        return np.array([[ev[k][j].elapsed_time(ev[k][j + 1]) for j in range(len(ev[k]) - 1)]
                         for k in range(K)])

    barrier()
    torch.cuda.synchronize()
    with ClockSampler(torch.cuda.current_device()) as clocks:
        steps_ms = timed_steps(False)
    barrier()
    elapsed = max_over_ranks(float(steps_ms.sum()) / 1e3)
    phase = timed_steps(True)  # the per-phase breakdown (same K steps again)
    barrier()
    t_mark, t_cap, t_write = phase.mean(axis=0) / 1e3

    nbytes, local, per_table, _, _ = ck.layout()
    dirty_rank = int(local.sum())
    dirty_all = int(per_table.sum())  # every rank's dirty rows (from the count all_gather)
    row_bytes = DIM * 4
    value = dirty_all * row_bytes * K / elapsed / 1e9
    _ = ck.fetch()  # error flags of the timed steps

    # ---- parity of the last timed step's payload at full scale (oracle as checker) ------
    look_host = [lk.cpu().numpy() for lk in lookups]
    parity, host_payload = None, None
    if args.verify_rows > 0:
        host_payload = ck.payload[:nbytes].cpu().numpy()
        parity = verify_step(ck, tables, look_host, w, host_payload, local, args.verify_rows)

    # roofline of the dominant kernel (algorithmic bytes / its mean duration)
    rec = ck.rec
    k1_bytes = stream.nbytes
    k3_bytes = dirty_rank * (row_bytes + 8 + rec) + len(cards) * 24
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured" if peaks else "fallback"
    phases = {
        "mark": {"ms": t_mark * 1e3, "bytes": k1_bytes, "GB/s": k1_bytes / t_mark / 1e9},
        "capture": {"ms": t_cap * 1e3},
        "write": {"ms": t_write * 1e3, "bytes": k3_bytes, "GB/s": k3_bytes / t_write / 1e9},
    }
    dom = "mark" if t_mark >= t_write else "write"
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(args.workload, {}).get(dom)
    wk = ("ds::writer_warp_kernel (adaptive greedy ranges, compute-bound)" if w["adaptive"]
          else "ds::writer_warp_kernel (naive ranges)")
    roofline = {"bound": "hbm", "kernel": {"mark": "ds::mark_tma_kernel", "write": wk}[dom],
                "measured_over": {"mark": "the mark phase (one mark_tma launch per step)",
                                  "write": "the write phase (one writer launch per step)"}[dom],
                "traffic_source": "profiles/traffic.json: dram read+write bytes per launch, "
                                  "ncu --set full",
                "achieved": phases[dom]["GB/s"], "peak": peak, "unit": "GB/s",
                "frac": phases[dom]["GB/s"] / peak, "traffic": traffic,
                "peak_source": peak_src}
    if traffic:
        # DRAM moves whole sectors: a dirty row narrower than the 128-byte
        # granule the L2 fetches for a random row read costs that granule, so
        # measured traffic above the algorithmic bytes is the rows' scatter,
        # not re-reads (C2: 64-byte rows)
        alg = phases[dom].get("bytes")  # per step = per launch
        roofline["traffic_vs_algorithmic"] = traffic / alg if alg else None
        roofline["traffic_note"] = (
            "ncu dram read+write bytes per launch / algorithmic bytes per launch; rows of "
            f"{4 * DIM} B at random addresses fetch whole L2 sectors (granule 128 B)")
    if w["adaptive"] and dom == "write":
        # the greedy search is compute-bound: SURVEY 8(d)'s op count per row,
        # 13*d*(E+1) + 2d with E = 2*steps + 1 candidate evaluations, against
        # the fp32 lane-op rate (SMs x 128 x max SM clock)
        bins, ratio = {2: (25, 0.5), 3: (25, 0.2), 4: (45, 0.2)}[w["bitwidth"]]
        E = 2 * int(np.floor(bins * ratio + 1e-9)) + 1
        ops = dirty_rank * (13 * DIM * (E + 1) + 2 * DIM)
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        peak_ops = sms * 128 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
        roofline["compute"] = {"unit": "Gop/s", "ops_per_step": ops, "achieved": ops / t_write / 1e9,
                               "peak": peak_ops / 1e9, "frac": ops / t_write / peak_ops,
                               "evaluations_per_row": E}

    # ---- stall-window staging (not in the metric) -------------------
    # the stall a training loop sees: K2 + the dirty-row gather; K3 then runs
    # from the staged copy on a side stream
    staged = None
    if True:
        cap = int(dirty_rank * 1.25) + 1024
        sst, stot = [], []
        for k in range(max(3, min(K, 20)) + 3):
            ck.mark(stream)
            flush.fill_(k & 0xFF)
            s0, s2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s0.record()
            stall_end = ck.checkpoint(staged_rows=cap)
            ck.wait()
            s2.record()
            torch.cuda.synchronize()
            if k >= 3:
                sst.append(s0.elapsed_time(stall_end))
                stot.append(s0.elapsed_time(s2))
        _ = ck.fetch()
        staged = {"stall_ms": float(np.median(sst)), "checkpoint_ms": float(np.median(stot)),
                  "direct_stall_ms": (t_cap + t_write) * 1e3,
                  "note": "stall = capture + dirty-row gather; K3 then runs from the copy on a "
                          "side stream (the direct path stalls for capture + K3)"}

    # ---- the store's payload checksum on device (not in the metric) ---------------------
    # (store.py:46-47 zlib.crc32 of every shard payload)
    crc = None
    if nbytes > 0:
        from paper_2010_08679_b200.payload import crc32 as ds_crc32
        crc_out = torch.empty(1, dtype=torch.int32, device=dev)
        for _ in range(3):
            ds_crc32(ck.payload, nbytes, out=crc_out)
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record()
        for _ in range(10):
            ds_crc32(ck.payload, nbytes, out=crc_out)
        c1.record()
        torch.cuda.synchronize()
        tc = c0.elapsed_time(c1) / 10 / 1e3
        crc = {"ms": tc * 1e3, "bytes": int(nbytes), "GB/s": nbytes / tc / 1e9,
               "note": "zlib.crc32 of the step's payload on device (L2-warm), outside the metric"}

    # ---- e2e through the public API with host buffers --------------------------------
    # The public pipeline API (paper_2010_08679_b200.pipeline): each step's
    # lookups come from pinned host memory (H2D) and each step's payload goes
    # back to pinned host memory (D2H); copies overlap the kernels of the
    # neighbouring steps on their own streams.  Timed on the host clock
    # (the pipeline synchronises on the host between steps).  Headline: the
    # lookups as a data loader emits them -- int32 row ids per table
    # (DirtyBitmap.mark's input, tracker.py:27-36), K1 = ds_mark over the
    # concatenation; secondary: the bit-packed LookupStream (packed on the
    # host once, outside the timed region).
    e2e = None
    if not args.no_e2e:
        from paper_2010_08679_b200.pipeline import CheckpointPipeline
        seg_off = np.concatenate([[0], np.cumsum([lk.size for lk in look_host])]).astype(np.int64)
        seg_tab = np.arange(len(look_host), dtype=np.int64)
        host_i32 = torch.from_numpy(np.concatenate(look_host).astype(np.int32)).pin_memory()

        def e2e_run(feed, cap, dtype, steps):
            pipe = CheckpointPipeline(ck, cap, dtype)
            for _ in range(3):
                feed(pipe)
            pipe.drain()
            h2d0, d2h0 = pipe.h2d_bytes, pipe.d2h_bytes
            barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for _ in range(steps):
                feed(pipe)
            pipe.drain()
            el = max_over_ranks(time.perf_counter() - t0)
            barrier()
            out = {"value": dirty_all * row_bytes * steps / el / 1e9, "unit": "GB/s",
                   "h2d_bytes_per_step": int((pipe.h2d_bytes - h2d0) / steps),
                   "d2h_bytes_per_step": int((pipe.d2h_bytes - d2h0) / steps),
                   "ms_per_step": el / steps * 1e3}
            ck.payload = pipe.payload[0]
            return out

        e2e = e2e_run(lambda p: p.submit(host_i32, seg_off, seg_tab), host_i32.numel(),
                      torch.int32, K)
        e2e.update(lookups="int32 row ids per table, pinned host memory (106 B per C2 batch "
                           "position of 26 lookups)" if args.workload == "C2" else
                           "int32 row ids per table, pinned host memory",
                   overlap="H2D(k+1) | kernels(k) | D2H(k-1) on separate streams")
        packed = e2e_run(lambda p: p.submit(host_stream), host_stream.nbytes, torch.uint8, K)
        packed["lookups"] = ("LookupStream: ids bit-packed at ceil(log2 rows) bits, packed on "
                             "the host outside the timed region")
        e2e["packed_stream"] = packed
        # the pipeline's own D2H'd payloads (double-buffered slots) of 3
        # consecutive steps are the verified payload, byte for byte
        if host_payload is not None:
            pipe = CheckpointPipeline(ck, host_i32.numel(), torch.int32, keep_outputs=True)
            for _ in range(3):
                pipe.submit(host_i32, seg_off, seg_tab)
            outs = pipe.drain()
            ck.payload = pipe.payload[0]
            same = sum(1 for o in outs if o == host_payload.tobytes())
            parity["pipeline_payloads_equal"] = f"{same}/{len(outs)}"
            if same != len(outs):
                parity["mismatches"] += len(outs) - same

    # ---- CPU baseline (rank 0, N == 1): oracle port on the same inputs ----------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        del lookups
        big = sum(t.values.numel() for t in tables) * 4 > (8 << 30)
        host_tables = None if big else [t.values.cpu().numpy() for t in tables]

        def fetch(t, ids):
            tv = tables[t].values
            return tv.index_select(0, torch.from_numpy(np.asarray(ids, np.int64)).to(dev)).cpu().numpy()

        c = cpu_measure(w, host_tables, look_host, shipped=not args.no_shipped,
                        payload=host_payload, fetch=fetch)
        cpu = {k: c[k] for k in ("value", "unit", "cores", "kind", "sample")}
        cpu["reference_as_shipped"] = c.get("reference_as_shipped")

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": elapsed / K * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic",
            "config": dict(workload_desc(w), dirty_rows_per_step=dirty_all,
                           parallelism=f"row-sharded x{world}", inputs=input_gen,
                           **({"rank_alignment": "device all_reduce after each untimed L2 flush"}
                              if world > 1 else {})),
            "l2_fetch_bytes": l2_fetch,
            "rows_per_s": dirty_all * K / elapsed,
            "roofline": roofline, "phases": phases, "payload_crc32": crc, "staged": staged,
            "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks.summary(),
            "parity": parity,
            # per timed step: mark_tma 1 + cap3_count 1 + cap3_emit 1 + writer 1 (the
            # layout, the count exchange and the error sum run inside the writer)
            "gpu_launches": K * 4,
            "payload_bytes_per_step": int(nbytes) if world == 1 else None,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def restore_launches(h, incremental):
    """ds_restore_payload launches engine.apply_payload makes for one payload:
    one per run of <= MAX_TABLES sections sharing (dim, bitwidth, aux)."""
    from paper_2010_08679_b200 import _lib
    from paper_2010_08679_b200.payload import parse_headers
    keys = [(i.dim, i.bitwidth, i.aux) for i in parse_headers(h, incremental)]
    n, k0 = 0, 0
    while k0 < len(keys):
        k1 = k0
        while k1 < len(keys) and k1 - k0 < _lib.MAX_TABLES and keys[k1] == keys[k0]:
            k1 += 1
        n, k0 = n + 1, k1
    return n


def run_restore(args):
    """C5: restore a 1 full + 5 incremental chain through the public API
    (engine.apply_payload: one ds_restore_payload launch per payload).

    One process per GPU; rank g restores rows [g*R/N, (g+1)*R/N) of every
    table (SURVEY 8(e) "Restore"), uploading only its rows' records
    (engine.rank_slices: a slice of the full section, a binary search over
    the sorted row column of each incremental one).  value: restored fp32
    row bytes of all ranks / max-over-ranks device time of the chain with the
    rank's slices resident in HBM; e2e: the same with the slices H2D-copied
    from pinned host memory inside the timed region.
    """
    import torch
    import torch.distributed as dist
    import paper_2010_08679_b200 as ds
    from paper_2010_08679_b200.engine import ShardWriter, apply_payload, rank_slices
    from paper_2010_08679_b200.payload import parse_headers
    from paper_2010_08679_b200.sharded import ShardedCheckpointer, shard_rows
    from paper_2010_08679_b200.tracker import ModelTracker

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group("nccl", device_id=dev)

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local_rank])

    w = workload_of(args)
    cards, dim = w["cards"], w["dim"]
    gen = torch.Generator(device=dev)
    gen.manual_seed(args.seed * 7919)  # every rank builds the same chain
    tables = [ds.DeviceTable(t, torch.rand((r, dim), generator=gen, device=dev).mul_(2).sub_(1))
              for t, r in enumerate(cards)]
    # the chain: a full checkpoint, then 5 intervals of Zipf lookups
    chain = []
    full = ShardWriter(tables, w["bitwidth"], adaptive=None, device=dev)
    buf = torch.empty(full.payload_bytes(None) + 16, dtype=torch.uint8, device=dev)
    full.write(buf)
    n, _ = full.finish()
    chain.append(("full", buf[:n].clone()))
    ck = ShardedCheckpointer(tables, w["bitwidth"], adaptive_overrides={w["bitwidth"]: None},
                             device=dev)
    for k in range(w["restore"]):
        lk = [lookups_torch(w["lookups"], r, w["n_per_table"], gen, dev) for r in cards]
        ck.step(pack_lookups(lk, cards, dev)[1])
        nb = int(ck.writer.sec_off[-1].item())
        chain.append(("incremental", ck.payload[:nb].clone()))
        for t in tables:  # the training step between checkpoints
            t.values.add_(0.01)
    host = [(kind, b.cpu().numpy().tobytes()) for kind, b in chain]
    del chain, ck, full, buf
    # this rank's rows of every table, and its slice of every payload
    ranges = {t: shard_rows(r, world, rank) for t, r in enumerate(cards)}
    out = {t: ds.DeviceTable(t, torch.zeros((hi - lo, dim), device=dev), row_base=lo,
                             total_rows=cards[t]) for t, (lo, hi) in ranges.items()}
    tr = ModelTracker({t: o.rows for t, o in out.items()}, device=dev)
    base = {tid: tr.baseline_bitmap(tid) for tid in out}
    slices = []
    for kind, h in host:
        infos = parse_headers(h, kind != "full")
        hs, descs = rank_slices(h, infos, kind != "full", [ranges[i.table_id] for i in infos])
        pin = torch.from_numpy(hs).pin_memory()
        slices.append((kind, h, pin, pin.to(dev), descs))
    rows_restored = sum(hi - lo for lo, hi in ranges.values())  # this rank's rows
    # records the chain restores (all ranks): every row of the full section
    # plus every incremental record -- each is unpacked, dequantized, scattered
    chain_records = sum(i.rows for kind, h in host for i in parse_headers(h, kind != "full"))
    chain_records_rank = sum(d[1] for kind, _, _, _, descs in slices for d in descs
                             if kind != "full") + rows_restored

    def restore_once(from_host):
        checks = []
        for kind, h, pin, dbuf, descs in slices:
            if from_host:
                dbuf.copy_(pin, non_blocking=True)
            checks.append(apply_payload(h, kind != "full", out, base if kind != "full" else None,
                                        device=dev, device_buf=dbuf, sync=False, slice_descs=descs))
        return checks

    for _ in range(max(3, args.warmup)):
        for c in restore_once(False):
            c()
    torch.cuda.synchronize()
    K = args.steps
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    times, times_e2e = [], []
    with ClockSampler(local_rank) as clocks:
        for k in range(K):
            flush.fill_(k & 0xFF)
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            checks = restore_once(False)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
            for c in checks:
                c()
        for k in range(K):
            barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            checks = restore_once(True)
            for c in checks:
                c()
            torch.cuda.synchronize()
            times_e2e.append(time.perf_counter() - t0)
    t = max_over_ranks(float(np.mean(times)))
    te = max_over_ranks(float(np.mean(times_e2e)))

    # parity: every restored row of this rank (and the rebuilt since-baseline
    # bits) against the CPU oracle applying the same chain (engine.py:459-485)
    parity = None
    if args.verify_rows > 0:
        from oracle import oracle as O
        t0 = time.perf_counter()
        split = [(kind != "full", dict(O.split_sections(h, kind != "full"))) for kind, h in host]
        rows_ok = rows_n = bits_bad = 0
        for tid, (lo, hi) in ranges.items():
            want = np.zeros((cards[tid], dim), np.float32)
            bits = np.zeros((cards[tid] + 7) // 8, np.uint8)
            for inc, secs in split:
                if tid in secs:
                    O.apply_section(secs[tid], inc, want, None, bits if inc else None)
            got = out[tid].values.cpu().numpy()
            rows_ok += int(np.all(got.view(np.uint32) == want[lo:hi].view(np.uint32), axis=1).sum())
            rows_n += hi - lo
            ref_bits = np.unpackbits(bits, bitorder="little")[:cards[tid]][lo:hi]
            got_bits = np.unpackbits(base[tid].to_bytes(), bitorder="little")[:hi - lo]
            bits_bad += int(not np.array_equal(ref_bits, got_bits))
        parity = {"rows_checked": rows_n, "mismatches": rows_n - rows_ok + bits_bad,
                  "baseline_bitmaps_checked": len(ranges),
                  "checked_against": "CPU oracle applying the same chain (every row of this "
                                     "rank's tables, bit-exact float32; since-baseline bits)",
                  "seconds": time.perf_counter() - t0}
        if world > 1:
            mm = torch.tensor([parity["mismatches"], rows_n], dtype=torch.int64, device=dev)
            dist.all_reduce(mm)
            parity["mismatches"], parity["rows_checked"] = int(mm[0].item()), int(mm[1].item())
    h2d = sum(p.numel() for _, _, p, _, _ in slices)
    full_bytes = sum(len(h) for _, h in host)
    nbytes = chain_records * dim * 4  # restored row bytes of all ranks
    # roofline: this rank's algorithmic bytes = its slices read + its restored
    # fp32 rows written (every record of the rank is applied once per payload)
    alg = h2d + chain_records_rank * dim * 4
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    peak = float(peaks.get("hbm_gbs", 6650.0))
    if rank == 0:
        line = {
            "metric": "restored GB/s of embedding rows (unpack+dequantize+scatter)",
            "value": nbytes / t / 1e9, "unit": "GB/s", "n_gpus": world, "steps": K,
            "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u8->f32 via f64",
            "data": "synthetic",
            "config": dict(workload_desc(w), chain_records=chain_records, chain_payload_bytes=full_bytes,
                           rank_upload_bytes=h2d, rows_per_rank=rows_restored,
                           parallelism=f"row-sharded x{world} (rank-local slices)",
                           timing="CUDA events at each chain's bounds, max over ranks"),
            "roofline": {"bound": "hbm",
                         "kernel": "ds::restore_payload_kernel (one launch per payload of the chain)",
                         "achieved": alg / t / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": alg / t / 1e9 / peak,
                         "traffic": (json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
                                     .get("C5", {}).get("restore_chain")
                                     if os.path.exists(os.path.join(ROOT, "profiles", "traffic.json"))
                                     else None),
                         "traffic_note": "dram read+write bytes of the chain's launches (ncu --set full), "
                                         "per chain"},
            "e2e": {"value": nbytes / te / 1e9, "unit": "GB/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": 4 * len(host) * len(cards)},
            "parity": parity,
            "clocks": clocks.summary(),
            "gpu_launches": K * sum(restore_launches(h, kind != "full") for (kind, h) in host),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse_args()
    if args.impl == "reference":
        run_reference(args)
    elif WORKLOADS[args.workload].get("restore"):
        run_restore(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

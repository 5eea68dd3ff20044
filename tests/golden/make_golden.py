"""Generate the golden fixtures by importing the reference `deltasnap` package.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports /root/reference/pkg/src read-only and writes small .npz fixtures
next to this script.  The fixtures travel with the repo; /root/reference does
not exist on the GPU box.  Every fixture records the numpy version it was
made with, because the reference's float64 results follow numpy's reduction
order.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))


def _ref():
    sys.dont_write_bytecode = True
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import deltasnap  # noqa: F401
    return deltasnap


def codec_fixture(ds):
    """quant.py:93-209,372-395 on the benchmark corpus (quant.py:418-438)."""
    q = ds.quant
    out = {"numpy_version": np.array(np.__version__)}
    for d in (1, 3, 7, 8, 9, 16, 33, 64, 65, 128, 130):
        x = q.benchmark_corpus(64, d, seed=d)
        # a constant row and a grid-valued row as edge cases
        x[0, :] = np.float32(0.375)
        x[1, :] = (np.arange(d, dtype=np.float32) % 5) * np.float32(0.25)
        out[f"x_d{d}"] = x
        lo, hi = x.min(axis=1), x.max(axis=1)
        for n in (2, 3, 4, 8):
            codes = q.quantize_rows(x, lo, hi, n)
            out[f"codes_d{d}_n{n}"] = codes
            out[f"deq_d{d}_n{n}"] = q.dequantize_rows(codes, lo, hi, n)
            out[f"me_d{d}_n{n}"] = q.reconstruction_errors(x, lo, hi, n)
            out[f"packed_d{d}_n{n}"] = q.pack_code_rows(codes, n)
            if n != 8:
                cfg = q.default_adaptive_config(n)
                amin, amax = q.adaptive_params_rows(x, n, cfg)
                out[f"amin_d{d}_n{n}"] = amin
                out[f"amax_d{d}_n{n}"] = amax
                acodes = q.quantize_rows(x, amin, amax, n)
                out[f"acodes_d{d}_n{n}"] = acodes
    # non-default search configs (tests/test_quant.py:206-216)
    rng = np.random.default_rng(5)
    x = rng.normal(0, 1, (30, 16)).astype(np.float32)
    x[:, 0] *= 10
    out["cfg_x"] = x
    for n in (2, 3, 4):
        for bins, ratio in ((25, 0.5), (25, 0.2), (45, 0.2), (10, 0.3), (2, 1.0), (1, 1.0)):
            amin, amax = q.adaptive_params_rows(x, n, q.AdaptiveConfig(bins, ratio))
            out[f"cfg_min_n{n}_b{bins}_r{ratio}"] = amin
            out[f"cfg_max_n{n}_b{bins}_r{ratio}"] = amax
    return out


def tracker_fixture(ds):
    """tracker.py:27-139: a mark/capture/reset sequence with both scopes."""
    rng = np.random.default_rng(11)
    rows = {0: 333, 1: 64, 2: 1000}
    tr = ds.ModelTracker(rows)
    out = {"numpy_version": np.array(np.__version__), "rows": np.array([333, 64, 1000])}
    step = 0
    for phase in range(3):
        for tid, r in rows.items():
            idx = rng.integers(0, r, size=int(rng.integers(0, 80)))
            out[f"mark_p{phase}_t{tid}"] = idx
            tr.mark(tid, idx)
        view = tr.capture()
        for tid in rows:
            out[f"int_p{phase}_t{tid}"] = view.interval_rows[tid]
            out[f"base_p{phase}_t{tid}"] = view.baseline_rows[tid]
        out[f"frac_p{phase}"] = np.array([view.interval_fraction, view.baseline_fraction])
        tr.reset_interval()
        step += 1
    return out


def payload_fixture(ds):
    """engine.py:118-189 build_shard_payload bytes for full/incremental plans."""
    from deltasnap.policy import CheckpointPlan
    out = {"numpy_version": np.array(np.__version__)}
    for aux in (False, True):
        cfg = ds.ModelConfig(num_tables=3, rows_per_table=300, dim=12, num_shards=2,
                             has_aux_state=aux, dense_dim=8)
        model = ds.init_model(cfg, 7)
        wl = ds.WorkloadConfig(model=cfg, batch_size=40, zipf_s=1.1, batches_per_interval=10,
                               num_intervals=2, seed=7)
        tr = ds.ModelTracker({t: cfg.rows_per_table for t in range(cfg.num_tables)})
        for _ in range(10):
            ds.apply_batch(model, tr, wl)
        snap = model.snapshot()
        view = tr.capture()
        tag = f"aux{int(aux)}"
        for t in range(cfg.num_tables):
            out[f"{tag}_values_t{t}"] = snap.tables[t].values
            if aux:
                out[f"{tag}_aux_t{t}"] = snap.tables[t].aux
            out[f"{tag}_rows_t{t}"] = view.baseline_rows[t]
        for bw in (None, 2, 3, 4, 8):
            for kind in ("full", "incremental"):
                plan = CheckpointPlan(kind=kind, rows=view.baseline_rows if kind == "incremental"
                                      else None, bitwidth=bw)
                for sid in range(cfg.num_shards):
                    for ov in (None, {4: ds.AdaptiveConfig(1, 0.5)}):
                        if ov is not None and bw != 4:
                            continue
                        blob, qr, err = ds.build_shard_payload(snap, plan, sid, 64, ov)
                        key = f"{tag}_bw{bw}_{kind}_s{sid}" + ("_naive4" if ov else "")
                        out[key] = np.frombuffer(blob, dtype=np.uint8)
                        out[key + "_meta"] = np.array([qr, err])
    return out


def restore_fixture(ds):
    """engine.py:443-512: a consecutive-increment chain (1 full + 5 deltas)."""
    out = {"numpy_version": np.array(np.__version__)}
    for bw in (None, 3, 8):
        cfg = ds.ModelConfig(num_tables=2, rows_per_table=200, dim=8, num_shards=2,
                             has_aux_state=True, dense_dim=4)
        wl = ds.WorkloadConfig(model=cfg, batch_size=30, zipf_s=1.1, batches_per_interval=5,
                               num_intervals=6, seed=3)
        model = ds.init_model(cfg, 3)
        tr = ds.ModelTracker({t: cfg.rows_per_table for t in range(cfg.num_tables)})
        cstore = ds.CheckpointStore(ds.InMemoryStore(), "g")
        eng = ds.CheckpointEngine(model, tr, cstore, ds.RunConfig(
            checkpoint_interval=5, policy="consecutive_increment", bitwidth=bw, chunk_rows=16,
            keep_last_n=10, workers=1))
        for _ in range(6):
            for _ in range(5):
                ds.apply_batch(model, tr, wl)
            eng.on_interval_end()
            eng.drain()
        eng.shutdown()
        restored = ds.restore(cstore)
        tag = f"bw{bw}"
        chain = [cstore.read_manifest(c) for c in restored.chain_ids]
        out[f"{tag}_nchain"] = np.array(len(chain))
        for i, m in enumerate(chain):
            out[f"{tag}_kind{i}"] = np.array(m.kind)
            for sid, entry in sorted(m.shards.items()):
                out[f"{tag}_m{i}_s{sid}"] = np.frombuffer(cstore.store.get(entry.key), np.uint8)
        for t in range(cfg.num_tables):
            out[f"{tag}_values_t{t}"] = restored.model.tables[t].values
            out[f"{tag}_aux_t{t}"] = restored.model.tables[t].aux
            out[f"{tag}_base_t{t}"] = restored.tracker.since_baseline(t).dirty_rows()[0]
    return out


def main():
    ds = _ref()
    for name, fn in (("codec", codec_fixture), ("tracker", tracker_fixture),
                     ("payload", payload_fixture), ("restore", restore_fixture)):
        path = os.path.join(HERE, f"{name}.npz")
        np.savez_compressed(path, **fn(ds))
        print(path, os.path.getsize(path))


if __name__ == "__main__":
    main()

"""restore() as a drop-in for the reference's (engine.py:415-535), and the
reference CheckpointEngine / sim.run driving this package's hot path.

The reference package is imported from its offline install (baseline/_ref,
which travels to the GPU box) -- as the caller whose stores and engine this
package plugs into, never as the thing measured.  Stores are written by the
unmodified reference engine; restores are compared field by field
(RestoredRun), by state_digest (model.py:156-165) and by the rebuilt
since-baseline bits (engine.py:476).
"""

import numpy as np
import pytest

from tests.conftest import import_reference_anywhere

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ds():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2010_08679_b200 as m
    return m


@pytest.fixture(scope="module")
def ref():
    return import_reference_anywhere()


def _workload(ref, rows=400, dim=8, tables=2, shards=2, intervals=6, aux=False):
    model = ref.ModelConfig(num_tables=tables, rows_per_table=rows, dim=dim, num_shards=shards,
                            dense_dim=16, has_aux_state=aux)
    return ref.WorkloadConfig(model=model, batch_size=60, zipf_s=1.1, batches_per_interval=5,
                              num_intervals=intervals, seed=3)


def _run_reference(ref, policy, bitwidth, keep=8, aux=False, schedule=None, intervals=6):
    store = ref.InMemoryStore()
    cfg = ref.RunConfig(checkpoint_interval=5, policy=policy, bitwidth=bitwidth, workers=2,
                        keep_last_n=keep)
    rep = ref.run(_workload(ref, aux=aux, intervals=intervals), cfg, store, schedule=schedule,
                  run_id="r")
    return store, ref.CheckpointStore(store, "r"), rep


def _errors(ds, ref, name):
    return (getattr(ds.errors, name), getattr(ref.errors, name))


def _same_restore(ds, ref, ours, want):
    assert ours.chain_ids == want.chain_ids
    assert ours.baseline_id == want.baseline_id
    assert ours.baseline_payload_bytes == want.baseline_payload_bytes
    assert ours.manifest.checkpoint_id == want.manifest.checkpoint_id
    assert ours.history.sizes == want.history.sizes
    assert ours.model.reader.batches_consumed == want.model.reader.batches_consumed
    assert ours.model.reader.rng_cursor == want.model.reader.rng_cursor
    assert ours.model.config.num_tables == want.model.config.num_tables
    assert ours.model.config.rows_per_table == want.model.config.rows_per_table
    assert ours.model.config.dim == want.model.config.dim
    assert ours.model.config.num_shards == want.model.config.num_shards
    assert ours.model.config.dense_dim == want.model.config.dense_dim
    assert ours.model.config.has_aux_state == want.model.config.has_aux_state
    # bit-identical tables, aux and dense (model.py:156-165)
    assert ds.state_digest(ours.model) == ref.state_digest(want.model)
    for tid, t in want.model.tables.items():
        got = ours.model.tables[tid].values.cpu().numpy()
        assert np.array_equal(got.view(np.uint32), t.values.view(np.uint32)), tid
        # since-baseline scope rebuilt at restore (engine.py:476)
        b_ours = ours.tracker.baseline_bitmap(tid).to_bytes()
        b_ref = want.tracker.since_baseline(tid)._words
        assert np.array_equal(b_ours, b_ref), tid


@pytest.mark.parametrize("policy,bitwidth,aux", [
    ("consecutive_increment", 8, False),
    ("consecutive_increment", 4, True),     # reference default: adaptive 4-bit
    ("one_shot_baseline", 3, False),
    ("intermittent", 2, False),
    ("full_only", None, False),             # fp32 sections
    ("one_shot_baseline", None, True),
])
def test_restore_every_checkpoint_matches_reference(ds, ref, policy, bitwidth, aux):
    _, cstore, _ = _run_reference(ref, policy, bitwidth, aux=aux)
    ids = cstore.valid_ids()
    assert ids
    for cid in ids:
        want = ref.engine.restore(cstore, checkpoint_id=cid)
        for on_dev in (False, True):
            ours = ds.restore(cstore, checkpoint_id=cid, verify_on_device=on_dev)
            _same_restore(ds, ref, ours, want)
    # newest valid checkpoint by default
    _same_restore(ds, ref, ds.restore(cstore), ref.engine.restore(cstore))


def _newest_shard_key(cstore):
    m = cstore.read_manifest(cstore.valid_ids()[-1])
    return m, sorted(m.shards.items())[0][1].key


@pytest.mark.parametrize("on_dev", (False, True))
def test_corrupt_shard_raises_and_falls_back(ds, ref, on_dev):
    store, cstore, _ = _run_reference(ref, "consecutive_increment", 8)
    m, key = _newest_shard_key(cstore)
    data = bytearray(store.get(key))
    data[len(data) // 2] ^= 0x40  # same size, wrong CRC32
    store.put(key, bytes(data))
    with pytest.raises(_errors(ds, ref, "IntegrityError")):
        ds.restore(cstore, verify_on_device=on_dev)
    with pytest.raises(_errors(ds, ref, "IntegrityError")):
        ref.engine.restore(cstore)
    ours = ds.restore(cstore, fallback=True, verify_on_device=on_dev)
    want = ref.engine.restore(cstore, fallback=True)
    assert ours.manifest.checkpoint_id < m.checkpoint_id
    _same_restore(ds, ref, ours, want)


@pytest.mark.parametrize("on_dev", (False, True))
def test_corrupt_dense_is_detected(ds, ref, on_dev):
    """store.verify checks the dense object's CRC32 too (store.py:491-501);
    the device-verified path checks it on the host."""
    store, cstore, _ = _run_reference(ref, "consecutive_increment", 8)
    m = cstore.read_manifest(cstore.valid_ids()[-1])
    data = bytearray(store.get(m.dense.key))
    data[0] ^= 0x01
    store.put(m.dense.key, bytes(data))
    with pytest.raises(_errors(ds, ref, "IntegrityError")):
        ds.restore(cstore, verify_on_device=on_dev)
    ours = ds.restore(cstore, fallback=True, verify_on_device=on_dev)
    _same_restore(ds, ref, ours, ref.engine.restore(cstore, fallback=True))


def test_missing_object_and_empty_store(ds, ref):
    store, cstore, _ = _run_reference(ref, "consecutive_increment", 8)
    m, key = _newest_shard_key(cstore)
    store.delete(key)
    for on_dev in (False, True):
        with pytest.raises(_errors(ds, ref, "IntegrityError")):
            ds.restore(cstore, checkpoint_id=m.checkpoint_id, verify_on_device=on_dev)
    empty = ref.CheckpointStore(ref.InMemoryStore(), "none")
    with pytest.raises(_errors(ds, ref, "IntegrityError")):
        ds.restore(empty)


def test_to_reference_resumes_the_reference_trainer(ds, ref):
    """RestoredRun.to_reference gives the reference's own RestoredRun over host
    copies: the reference CheckpointEngine resumes from it."""
    _, cstore, _ = _run_reference(ref, "consecutive_increment", 4)
    want = ref.engine.restore(cstore)
    for kind in ("device", "reference"):
        got = ds.restore(cstore).to_reference(ref, tracker=kind)
        assert isinstance(got, ref.engine.RestoredRun)
        assert ref.state_digest(got.model) == ref.state_digest(want.model)
        assert got.history.sizes == want.history.sizes
        if kind == "reference":
            for tid in want.model.tables:
                assert np.array_equal(got.tracker.since_baseline(tid)._words,
                                      want.tracker.since_baseline(tid)._words)


def _substitute(monkeypatch, ds, ref):
    """What INTEGRATION.md tells a maintainer to bind: the writer, the
    tracker and restore of the reference engine/simulator replaced by this
    package's (the rest -- store, policy, threads -- stays the reference's)."""
    monkeypatch.setattr(ref.engine, "build_shard_payload", ds.build_shard_payload)
    monkeypatch.setattr(ref.sim, "ModelTracker", ds.ModelTracker)

    def engine_restore(cstore, *, fallback=False, checkpoint_id=None):
        return ds.restore(cstore, fallback=fallback,
                          checkpoint_id=checkpoint_id).to_reference(ref)

    monkeypatch.setattr(ref.sim, "engine_restore", engine_restore)


def _store_objects(store):
    return {k: store.get(k) for k in store.list("")}


@pytest.mark.parametrize("policy,bitwidth", [("consecutive_increment", 8),
                                             ("intermittent", 4),
                                             ("one_shot_baseline", 2)])
def test_reference_engine_with_this_hot_path(ds, ref, monkeypatch, policy, bitwidth):
    """sim.run (sim.py:283-352) with two trainer deaths: stock reference vs the
    reference with this package's tracker, writer and restore.  Every shard
    and dense object is byte-identical, manifests agree (quant_mean_l2 to
    1e-9: err_sum's summation order, engine.py:171-173), and so do the
    metrics and the surviving model."""
    sched = ref.FailureSchedule(((2, 3), (4, 1)))
    w = _workload(ref)
    cfg = ref.RunConfig(checkpoint_interval=5, policy=policy, bitwidth=bitwidth, workers=2,
                        keep_last_n=8)
    s_ref = ref.InMemoryStore()
    rep_ref, model_ref = ref.run(w, cfg, s_ref, schedule=sched, run_id="r",
                                 return_final_model=True)
    with monkeypatch.context() as mp:
        _substitute(mp, ds, ref)
        s_ours = ref.InMemoryStore()
        rep_ours, model_ours = ref.run(w, cfg, s_ours, schedule=sched, run_id="r",
                                       return_final_model=True)
    a, b = _store_objects(s_ref), _store_objects(s_ours)
    assert sorted(a) == sorted(b)
    import json
    for k in a:
        if k.endswith("manifest.json"):
            ja, jb = json.loads(a[k]), json.loads(b[k])
            qa, qb = ja.pop("quant_mean_l2"), jb.pop("quant_mean_l2")
            assert ja == jb, k
            assert (qa is None) == (qb is None)
            if qa is not None:
                assert abs(qa - qb) <= 1e-9 * max(abs(qa), 1e-30), k
        else:
            assert a[k] == b[k], k
    da, db = rep_ref.deterministic_view(), rep_ours.deterministic_view()
    for d in (da, db):
        d.pop("cumulative_restore_l2", None)
        d.pop("overruns", None)  # thread timing: a slower/faster writer, same outcome
        for r in d["intervals"]:
            r.pop("quant_mean_l2", None)
            r.pop("stall_seconds", None)
            r.pop("write_seconds", None)
    assert da == db
    assert rep_ref.resumes == rep_ours.resumes == 2
    assert abs(rep_ref.cumulative_restore_l2 - rep_ours.cumulative_restore_l2) <= \
        1e-9 * max(1.0, abs(rep_ref.cumulative_restore_l2))
    assert ref.state_digest(model_ref) == ref.state_digest(model_ours)

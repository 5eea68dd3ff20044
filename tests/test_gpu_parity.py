"""GPU parity: the sm_100a path against the reference's golden fixtures and
against the CPU oracle (bit-exact for ids, codes, params, bytes and restored
float32 tables; err_sum within 1e-12 relative, see engine.py docstring)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

DIMS = (1, 3, 7, 8, 9, 16, 33, 64, 65, 128, 130)


@pytest.fixture(scope="module")
def ds():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2010_08679_b200 as m
    return m


@pytest.fixture(scope="module")
def O():
    from oracle import oracle
    return oracle


def u32(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


def params_equal(a, b):
    """float32 equality with +0 == -0 (the documented signed-zero exception)."""
    return np.array_equal(np.asarray(a, np.float32), np.asarray(b, np.float32))


# --- codec ------------------------------------------------------------------------

@pytest.mark.parametrize("d", DIMS)
@pytest.mark.parametrize("n", (2, 3, 4, 8))
def test_codec_rows_match_golden(ds, golden, d, n):
    g = golden("codec")
    x = g[f"x_d{d}"]
    lo, hi = ds.quant.row_minmax(x)
    assert params_equal(lo, x.min(axis=1)) and params_equal(hi, x.max(axis=1))
    codes = ds.quantize_rows(x, lo, hi, n)
    assert np.array_equal(codes, g[f"codes_d{d}_n{n}"])
    deq = ds.dequantize_rows(codes, lo, hi, n)
    assert np.array_equal(u32(deq), u32(g[f"deq_d{d}_n{n}"]))
    me = ds.reconstruction_errors(x, lo, hi, n)
    assert np.array_equal(me.view(np.uint64), g[f"me_d{d}_n{n}"].view(np.uint64))
    packed = ds.pack_code_rows(codes, n)
    assert np.array_equal(packed, g[f"packed_d{d}_n{n}"])
    assert np.array_equal(ds.unpack_code_rows(packed, n, d), codes)
    if n != 8:
        cfg = ds.default_adaptive_config(n)
        amin, amax = ds.adaptive_params_rows(x, n, cfg)
        assert np.array_equal(amin, g[f"amin_d{d}_n{n}"])
        assert np.array_equal(amax, g[f"amax_d{d}_n{n}"])


@pytest.mark.parametrize("n", (2, 3, 4))
@pytest.mark.parametrize("bins,ratio", [(25, 0.5), (25, 0.2), (45, 0.2), (10, 0.3), (2, 1.0),
                                        (1, 1.0)])
def test_greedy_configs_match_golden(ds, golden, n, bins, ratio):
    g = golden("codec")
    amin, amax = ds.adaptive_params_rows(g["cfg_x"], n, ds.AdaptiveConfig(bins, ratio))
    assert np.array_equal(amin, g[f"cfg_min_n{n}_b{bins}_r{ratio}"])
    assert np.array_equal(amax, g[f"cfg_max_n{n}_b{bins}_r{ratio}"])


def test_known_answers(ds):
    assert ds.pack_codes([0, 1, 2, 3], 2) == b"\xe4"
    p = ds.QuantParams(2, 0.0, 3.0)
    assert ds.quantize(np.array([0.5, 1.5, 2.5], np.float32), p).codes.tolist() == [1, 2, 3]
    x = np.array([-1.0, 0.0, 2.0], np.float32)
    qv = ds.quantize(x, ds.uniform_params(x, 2))
    assert qv.codes.tolist() == [0, 1, 3]
    assert np.array_equal(ds.dequantize(qv), x)
    c = np.full(9, 0.123, np.float32)
    qv = ds.quantize(c, ds.uniform_params(c, 3))
    assert not qv.codes.any() and np.array_equal(ds.dequantize(qv), c)
    assert ds.quantize(np.array([-5.0, 5.0], np.float32),
                       ds.QuantParams(4, -1.0, 1.0)).codes.tolist() == [0, 15]
    with pytest.raises(ds.FormatError):
        ds.unpack_codes(b"\xc0", 2, 3)
    with pytest.raises(ds.FormatError):
        ds.unpack_codes(b"\x00\x00", 2, 3)
    with pytest.raises(ds.DataError):
        ds.pack_codes([4], 2)
    with pytest.raises(ds.FormatError):
        ds.dequantize_rows(np.array([[0, 4]], np.uint8), np.zeros(1, np.float32),
                           np.ones(1, np.float32), 2)
    with pytest.raises(ds.DataError):
        ds.adaptive_params_rows(np.array([[1.0, np.nan]], np.float32), 2,
                                ds.default_adaptive_config(2))
    with pytest.raises(ds.ConfigError):
        ds.quantize_rows(np.zeros((1, 2), np.float32), np.zeros(1, np.float32),
                         np.ones(1, np.float32), 5)


def _edge_rows(d, rng):
    rows = []
    rows.append(np.full(d, 0.375, np.float32))                       # constant
    rows.append((np.arange(d) % 5).astype(np.float32) * 0.25)        # grid: exact ties
    rows.append((np.arange(d) % 3).astype(np.float32) - 1.0)         # symmetric grid
    z = rng.normal(0, 1, d).astype(np.float32)
    z[0] = -0.0
    z[-1] = 0.0
    rows.append(z)                                                    # signed zeros
    o = rng.normal(0, 0.01, d).astype(np.float32)
    o[d // 2] = 50.0
    rows.append(o)                                                    # outlier
    rows.append((rng.normal(0, 1, d) * 1e-30).astype(np.float32))     # tiny range
    rows.append((rng.normal(0, 1, d) * 1e30).astype(np.float32))      # huge range
    rows.append((rng.normal(1000, 1e-3, d)).astype(np.float32))       # offset >> range
    rows.append(np.float32(rng.integers(-8, 8, d)) / 8)               # coarse grid
    return np.stack(rows)


@pytest.mark.parametrize("d", (1, 2, 5, 16, 31, 64, 128, 200, 1024))
@pytest.mark.parametrize("n", (2, 3, 4, 8))
def test_codec_edge_rows_vs_oracle(ds, O, d, n):
    rng = np.random.default_rng(d * 10 + n)
    x = np.concatenate([_edge_rows(d, rng),
                        (rng.normal(0, 1, (300, d)) * rng.lognormal(0, 2, (300, 1))).astype(
                            np.float32)])
    lo, hi = O.row_minmax(x)
    assert np.array_equal(ds.quantize_rows(x, lo, hi, n), O.quantize_rows(x, lo, hi, n))
    assert np.array_equal(ds.reconstruction_errors(x, lo, hi, n),
                          O.reconstruction_errors(x, lo, hi, n))
    if n != 8:
        bins, ratio = {2: (25, 0.5), 3: (25, 0.2), 4: (45, 0.2)}[n]
        a = ds.adaptive_params_rows(x, n, ds.AdaptiveConfig(bins, ratio))
        b = O.adaptive_params_rows(x, n, bins, ratio)
        assert params_equal(a[0], b[0]) and params_equal(a[1], b[1])


def test_adaptive_large_random_vs_oracle(ds, O):
    """200k rows x 64 from the reference's benchmark distribution (quant.py:418-438)."""
    rng = np.random.default_rng(42)
    n, d = 200_000, 64
    scale = np.exp(rng.normal(0, 1, n))
    x = (rng.normal(0, 1, (n, d)) * scale[:, None] + (rng.normal(0.4, 0.3, n) * scale)[:, None])
    cols = rng.integers(0, d, (n, 2))
    x[np.arange(n)[:, None], cols] += rng.choice([-1, 1], (n, 2)) * rng.uniform(4, 8, (n, 2)) * \
        scale[:, None]
    x = x.astype(np.float32)
    for nb in (2, 4):
        bins, ratio = {2: (25, 0.5), 4: (45, 0.2)}[nb]
        stats = torch.zeros(4, dtype=torch.int64, device="cuda")
        xd = torch.from_numpy(x).cuda()
        a = ds.adaptive_params_rows(xd, nb, ds.AdaptiveConfig(bins, ratio), stats=stats)
        b = O.adaptive_params_rows(x, nb, bins, ratio, nthreads=8)
        assert np.array_equal(a[0].cpu().numpy(), b[0]) and np.array_equal(a[1].cpu().numpy(), b[1])
        # the certified fast path decides almost everything in fp32
        assert int(stats[0]) < 0.05 * n * 2 * (bins * ratio), int(stats[0])


# --- tracker ---------------------------------------------------------------------

def test_tracker_matches_golden(ds, golden):
    g = golden("tracker")
    rows = [int(r) for r in g["rows"]]
    tr = ds.ModelTracker({t: r for t, r in enumerate(rows)})
    for phase in range(3):
        for t in range(len(rows)):
            tr.mark(t, g[f"mark_p{phase}_t{t}"])
        view = tr.capture()
        for t in range(len(rows)):
            assert np.array_equal(view.interval_rows[t], g[f"int_p{phase}_t{t}"])
            assert np.array_equal(view.baseline_rows[t], g[f"base_p{phase}_t{t}"])
        assert [view.interval_fraction, view.baseline_fraction] == g[f"frac_p{phase}"].tolist()
        tr.reset_interval()


def test_bitmap_semantics(ds):
    bm = ds.DirtyBitmap(0, 1000)
    assert bm.nbytes == 125
    assert ds.DirtyBitmap(0, 9).nbytes == 2
    bm.mark([3, 3, 3, 7, 999])
    assert bm.popcount() == 3
    assert bm.dirty_rows()[0].tolist() == [3, 7, 999]
    with pytest.raises(ds.BoundsError):
        bm.mark([1000])
    with pytest.raises(IndexError):
        bm.mark([-1])
    assert bm.popcount() == 3
    with pytest.raises(ds.ShapeError):
        bm.merge_or(ds.DirtyBitmap(0, 999))
    with pytest.raises(ds.ShapeError):
        bm.merge_or(ds.DirtyBitmap(1, 1000))
    other = ds.DirtyBitmap(0, 1000)
    other.mark([5, 7])
    u = bm.merge_or(other)
    assert u.dirty_rows()[0].tolist() == [3, 5, 7, 999]
    assert bm.dirty_rows()[0].tolist() == [3, 7, 999]
    ref_bytes = np.zeros(125, np.uint8)
    for r in (3, 5, 7, 999):
        ref_bytes[r >> 3] |= 1 << (r & 7)
    assert np.array_equal(u.to_bytes(), ref_bytes)
    # device-tensor marks: deferred BoundsError at the next sync point
    bm2 = ds.DirtyBitmap(0, 10)
    bm2.mark(torch.tensor([1, 10], device="cuda"))
    with pytest.raises(ds.BoundsError):
        bm2.popcount()
    tr = ds.ModelTracker({0: 8000, 1: 8000})
    assert tr.nbytes() == 4 * 1000


def test_merge_in_and_scope_resets(ds, O):
    """merge_in (tracker.py:46-49), reset_interval / reset_baseline
    (tracker.py:120-130) and mark_baseline (:132-134) against set semantics,
    and capture_device/capture_into with fold=1 (reset_interval) and fold=2
    (reset_baseline) in the same pass (engine.py:278-280)."""
    a, b = ds.DirtyBitmap(4, 100_000), ds.DirtyBitmap(4, 100_000)
    a.mark([1, 5, 99_999])
    b.mark([5, 6, 70_000])
    a.merge_in(b)
    assert a.dirty_rows()[0].tolist() == [1, 5, 6, 70_000, 99_999]
    assert b.dirty_rows()[0].tolist() == [5, 6, 70_000]  # the argument is untouched
    with pytest.raises(ds.ShapeError):
        a.merge_in(ds.DirtyBitmap(4, 99_999))
    with pytest.raises(ds.ShapeError):
        a.merge_in(ds.DirtyBitmap(5, 100_000))

    rng = np.random.default_rng(5)
    rows = {0: 1_000_003, 1: 70_001, 2: 17}
    for path in ("host", "capture_device", "capture_into"):
        tr = ds.ModelTracker(rows)
        ref_i = {t: set() for t in rows}
        ref_b = {t: set() for t in rows}
        for phase, fold in enumerate((1, 1, 2, 1, 2, 0)):
            for t, r in rows.items():
                idx = rng.integers(0, r, size=min(3 * r, 50_000))
                tr.mark(t, idx)
                ref_i[t] |= set(idx.tolist())
            if phase == 3:  # restore-time rebuild of the baseline scope
                extra = {t: rng.integers(0, r, 100) for t, r in rows.items()}
                for t in rows:
                    tr.mark_baseline(t, extra[t])
                    ref_b[t] |= set(extra[t].tolist())
            want_i = {t: np.array(sorted(ref_i[t]), np.int64) for t in rows}
            want_u = {t: np.array(sorted(ref_i[t] | ref_b[t]), np.int64) for t in rows}
            if path == "host":
                view = tr.capture()
                got_i, got_u = view.interval_rows, view.baseline_rows
                if fold == 1:
                    tr.reset_interval()
                elif fold == 2:
                    tr.reset_baseline()
            elif path == "capture_device":
                iv, uv = tr.capture_device(fold=fold)
                got_i = {t: iv[t].cpu().numpy() for t in rows}
                got_u = {t: uv[t].cpu().numpy() for t in rows}
            else:
                total = sum(rows.values())
                ids_i = torch.empty(total, dtype=torch.int64, device="cuda")
                ids_u = torch.empty(total, dtype=torch.int64, device="cuda")
                ci = torch.zeros(len(rows) + 1, dtype=torch.int64, device="cuda")
                cu = torch.zeros(len(rows) + 1, dtype=torch.int64, device="cuda")
                tr.capture_into(ids_u, cu, fold=0, scope="baseline")
                tr.capture_into(ids_i, ci, fold=fold, scope="interval")
                ci, cu = ci.cpu().numpy(), cu.cpu().numpy()
                assert ci[-1] == ci[:-1].sum() and cu[-1] == cu[:-1].sum()
                oi = np.concatenate([[0], np.cumsum(ci[:-1])])
                ou = np.concatenate([[0], np.cumsum(cu[:-1])])
                hi, hu = ids_i.cpu().numpy(), ids_u.cpu().numpy()
                got_i = {t: hi[oi[k]:oi[k] + ci[k]] for k, t in enumerate(rows)}
                got_u = {t: hu[ou[k]:ou[k] + cu[k]] for k, t in enumerate(rows)}
            for t in rows:
                assert np.array_equal(got_i[t], want_i[t]), (path, phase, t)
                assert np.array_equal(got_u[t], want_u[t]), (path, phase, t)
            if fold == 1:
                for t in rows:
                    ref_b[t] |= ref_i[t]
                    ref_i[t] = set()
            elif fold == 2:
                for t in rows:
                    ref_b[t], ref_i[t] = set(), set()
            for t in rows:
                assert np.array_equal(tr.interval_bitmap(t).dirty_rows()[0],
                                      np.array(sorted(ref_i[t]), np.int64)), (path, phase)
                assert np.array_equal(tr.baseline_bitmap(t).dirty_rows()[0],
                                      np.array(sorted(ref_b[t]), np.int64)), (path, phase)


def test_capture_large_vs_oracle(ds, O):
    rng = np.random.default_rng(1)
    rows = {0: 3_000_000, 1: 65_537, 2: 1, 3: 1_000_003}
    tr = ds.ModelTracker(rows)
    ref_i = {t: np.zeros((r + 7) // 8, np.uint8) for t, r in rows.items()}
    ref_b = {t: np.zeros((r + 7) // 8, np.uint8) for t, r in rows.items()}
    for phase in range(2):
        for t, r in rows.items():
            idx = rng.integers(0, r, size=min(r * 2, 400_000))
            tr.mark(t, idx)
            O.mark(ref_i[t], r, idx)
        view = tr.capture()
        for t, r in rows.items():
            assert np.array_equal(view.interval_rows[t], O.dirty_rows(ref_i[t], r))
            assert np.array_equal(view.baseline_rows[t], O.dirty_rows(ref_i[t] | ref_b[t], r))
            assert np.array_equal(tr.interval_bitmap(t).to_bytes(), ref_i[t])
        tr.reset_interval()
        for t in rows:
            ref_b[t] |= ref_i[t]
            ref_i[t][:] = 0


def test_mark_batch_multi_table(ds, O):
    rng = np.random.default_rng(3)
    rows = {t: int(r) for t, r in enumerate(rng.integers(1, 200_000, 26))}
    tr = ds.ModelTracker(rows)
    idx, seg = [], [0]
    for t, r in rows.items():
        a = rng.integers(0, r, 5000)
        idx.append(a)
        seg.append(seg[-1] + a.size)
    tr.mark_batch(torch.from_numpy(np.concatenate(idx)).cuda(), np.array(seg),
                  np.array(list(rows)))
    view = tr.capture()
    for k, (t, r) in enumerate(rows.items()):
        assert np.array_equal(view.interval_rows[t], np.unique(idx[k]))


@pytest.mark.parametrize("dtype", (torch.int32, torch.int64))
def test_mark_batch_table_kinds_and_bounds(ds, dtype):
    """Every per-table K1 form (shared byte map <= 65504 rows, shared bit
    window <= 524288 rows, cache + RED above), boundary sizes, Zipf-like
    repeats, ragged segment tails; out-of-range ids raise BoundsError at the
    next sync and never leak a bit (the byte map's dummy byte at `rows`)."""
    rng = np.random.default_rng(11)
    sizes = [1, 31, 32, 33, 1000, 16351, 16352, 16353, 65503, 65504, 65505, 65536, 65537,
             300_001, 524_287, 524_288, 524_289, 3_000_001]
    rows = {t: r for t, r in enumerate(sizes)}
    tr = ds.ModelTracker(rows)

    def batch(bad=False):
        idx, seg = [], [0]
        for t, r in rows.items():
            n = int(rng.integers(1, 40_000))
            hot = rng.integers(0, r, 8)
            a = np.where(rng.random(n) < 0.7, hot[rng.integers(0, 8, n)], rng.integers(0, r, n))
            if bad and t % 3 == 0:
                a[int(rng.integers(0, n))] = r if t % 2 == 0 else -1
            idx.append(a)
            seg.append(seg[-1] + a.size)
        return idx, seg

    idx, seg = batch()
    tr.mark_batch(torch.from_numpy(np.concatenate(idx)).to(dtype).cuda(), np.array(seg),
                  np.array(list(rows)))
    view = tr.capture()
    for k, t in enumerate(rows):
        assert np.array_equal(view.interval_rows[t], np.unique(idx[k])), t
    tr.reset_interval()
    idx, seg = batch(bad=True)
    tr.mark_batch(torch.from_numpy(np.concatenate(idx)).to(dtype).cuda(), np.array(seg),
                  np.array(list(rows)))
    with pytest.raises(ds.BoundsError):
        tr.capture()
    view = tr.capture()  # the valid ids of the batch are marked, nothing else
    for k, (t, r) in enumerate(rows.items()):
        good = idx[k][(idx[k] >= 0) & (idx[k] < r)]
        assert np.array_equal(view.interval_rows[t], np.unique(good)), t


# --- writer ------------------------------------------------------------------------

class _Snap:
    def __init__(self, tables, nshards):
        self.tables = tables
        self.nshards = nshards

    def shard_tables(self, sid):
        return [self.tables[t] for t in sorted(self.tables) if t % self.nshards == sid]


class _Tab:
    def __init__(self, tid, values, aux=None):
        self.table_id, self.values, self.aux = tid, values, aux


class _Plan:
    def __init__(self, kind, rows, bitwidth):
        self.kind, self.rows, self.bitwidth = kind, rows, bitwidth


@pytest.mark.parametrize("aux", (0, 1))
@pytest.mark.parametrize("bw", (None, 2, 3, 4, 8))
@pytest.mark.parametrize("kind", ("full", "incremental"))
def test_payload_matches_golden(ds, golden, aux, bw, kind):
    g = golden("payload")
    tag = f"aux{aux}"
    tabs = {t: _Tab(t, g[f"{tag}_values_t{t}"], g[f"{tag}_aux_t{t}"] if aux else None)
            for t in range(3)}
    rows = {t: g[f"{tag}_rows_t{t}"] for t in range(3)}
    snap = _Snap(tabs, 2)
    plan = _Plan(kind, rows if kind == "incremental" else None, bw)
    for sid in range(2):
        variants = [(None, "")] + ([({4: ds.AdaptiveConfig(1, 0.5)}, "_naive4")] if bw == 4 else [])
        for ov, suffix in variants:
            key = f"{tag}_bw{bw}_{kind}_s{sid}{suffix}"
            blob, qr, err = ds.build_shard_payload(snap, plan, sid, 64, ov)
            assert blob == g[key].tobytes(), key
            want_q, want_err = g[key + "_meta"]
            assert qr == want_q
            assert err == pytest.approx(want_err, rel=1e-12, abs=0)


@pytest.mark.parametrize("d", (1, 3, 8, 16, 20, 64, 100, 128, 256))
@pytest.mark.parametrize("bw", (None, 2, 3, 4, 8))
def test_payload_dims_vs_oracle(ds, O, d, bw):
    rng = np.random.default_rng(d + (bw or 0))
    rows = 3000
    tabs = {t: _Tab(t, (rng.normal(0, 1, (rows, d)) * rng.lognormal(0, 1, (rows, 1))).astype(
        np.float32), rng.random((rows, d)).astype(np.float32) if t == 1 else None)
        for t in range(3)}
    tabs[1].aux = None
    sel = {t: np.sort(rng.choice(rows, rng.integers(0, rows), replace=False)) for t in range(3)}
    sel[2] = np.zeros(0, np.int64)  # a 0-row table still gets its header
    for kind in ("incremental", "full"):
        plan = _Plan(kind, sel if kind == "incremental" else None, bw)
        blob, qr, err = ds.build_shard_payload(_Snap(tabs, 1), plan, 0)
        ref, qr_ref, err_ref = O.build_shard_payload(
            {t: (tabs[t].values, None) for t in tabs}, kind, sel, bw, [0, 1, 2], nthreads=8)
        assert blob == ref
        assert qr == qr_ref
        assert err == pytest.approx(err_ref, rel=1e-12, abs=1e-300)


def _near_tie_rows(rng, rows, d, L):
    """Rows whose fp32 code product t*inv rounds to exactly k + 1/2 while the
    exact product does not (t = RN(x - lo), inv = RN(RN(1/(hi - lo)) * L)):
    the fused (FFMA) and the rounded code of such an element can differ, and
    the reference's f64 code decides.  Found on the T workload (row 116128029:
    v_ref = 13.500000137), kept here as a constructed regression."""
    f32 = np.float32
    out = np.empty((rows, d), f32)
    for i in range(rows):
        lo = f32(-1 + rng.uniform(0, 0.1))
        hi = f32(1 - rng.uniform(0, 0.1))
        x = rng.uniform(lo, hi, d).astype(f32)
        x[0], x[1] = lo, hi
        inv = f32(f32(f32(1) / f32(hi - lo)) * f32(L))
        j = 2
        for k in rng.permutation(L)[: min(L, 24)]:
            x0 = f32(lo + f32((k + 0.5) / float(inv)))
            for s in range(-8, 9):
                xc = np.nextafter(x0, f32(np.inf if s > 0 else -np.inf), dtype=f32) if s else x0
                for _ in range(abs(s) - 1):
                    xc = np.nextafter(xc, f32(np.inf if s > 0 else -np.inf), dtype=f32)
                t = f32(xc - lo)
                p = float(t) * float(inv)  # exact: 24 x 24 bits
                if f32(p) == f32(k + 0.5) and p != k + 0.5 and lo < xc < hi and j < d:
                    x[j] = xc
                    j += 1
        out[i] = x
    return out


@pytest.mark.parametrize("bw", (2, 4, 8))
def test_writer_near_tie_products_vs_oracle(ds, O, bw):
    """Codes whose fp32 product rounds onto a tie (the packed writer fuses the
    product, its fixup pass must mirror exactly that arithmetic)."""
    rng = np.random.default_rng(77 + bw)
    d, rows = 128, 600
    x = _near_tie_rows(rng, rows, d, (1 << bw) - 1)
    tabs = {0: _Tab(0, x)}
    sel = {0: np.arange(0, rows, 3, dtype=np.int64)}
    ov = {bw: ds.AdaptiveConfig(1, 0.5)}  # naive ranges also at 2/4 bits
    for kind in ("incremental", "full"):
        plan = _Plan(kind, sel if kind == "incremental" else None, bw)
        blob, qr, err = ds.build_shard_payload(_Snap(tabs, 1), plan, 0, 1024, ov)
        ref, qr_ref, err_ref = O.build_shard_payload({0: (x, None)}, kind, sel, bw, [0],
                                                     adaptive={bw: (1, 0.5)}, nthreads=8)
        assert blob == ref
        assert err == pytest.approx(err_ref, rel=1e-12, abs=1e-300)


@pytest.mark.parametrize("bw", (2, 3, 4, 8))
@pytest.mark.parametrize("d", (16, 20, 128))
def test_writer_tie_heavy_rows_vs_oracle(ds, O, bw, d):
    """Grid-valued rows put many codes exactly on ties: every one of them goes
    through the exact-f64 fixup pass and must still match bit for bit."""
    rng = np.random.default_rng(bw * 100 + d)
    rows = 4000
    grid = rng.integers(-64, 64, (rows, d)).astype(np.float32) / np.float32(8)
    grid[::3] = (np.arange(d) % 7).astype(np.float32) * np.float32(0.5)  # exact half-steps
    grid[1::5] *= np.float32(1e-3)
    tabs = {0: _Tab(0, grid)}
    sel = {0: np.arange(0, rows, 2, dtype=np.int64)}
    for kind in ("incremental", "full"):
        plan = _Plan(kind, sel if kind == "incremental" else None, bw)
        ov = {bw: ds.AdaptiveConfig(1, 0.5)}  # naive ranges also at 2/3/4 bits
        blob, qr, err = ds.build_shard_payload(_Snap(tabs, 1), plan, 0, 1024, ov)
        ref, qr_ref, err_ref = O.build_shard_payload({0: (grid, None)}, kind, sel, bw, [0],
                                                     adaptive={bw: (1, 0.5)}, nthreads=8)
        assert blob == ref
        assert err == pytest.approx(err_ref, rel=1e-12, abs=1e-300)


@pytest.mark.parametrize("bw", (2, 8))
def test_writer_extreme_range_rows_vs_oracle(ds, O, bw):
    """Rows whose range leaves fp32's comfort zone (huge, tiny, subnormal)
    take the exact path for every code and for their error term."""
    rng = np.random.default_rng(7 + bw)
    rows, d = 600, 16
    x = rng.standard_normal((rows, d)).astype(np.float32)
    x[0::6] *= np.float32(1e37)
    x[1::6, :8] = np.float32(-3.0e38)
    x[1::6, 8:] = np.float32(3.0e38)
    x[2::6] = np.float32(1.0) + x[2::6] * np.float32(1e-33)
    x[3::6] *= np.float32(1e-40)  # subnormal
    x[4::6] = np.float32(5.0)  # constant rows
    tabs = {0: _Tab(0, x)}
    blob, qr, err = ds.build_shard_payload(_Snap(tabs, 1), _Plan("full", None, bw), 0, 1024,
                                           {bw: ds.AdaptiveConfig(1, 0.5)})
    ref, qr_ref, err_ref = O.build_shard_payload({0: (x, None)}, "full", None, bw, [0],
                                                 adaptive={bw: (1, 0.5)}, nthreads=8)
    assert blob == ref
    assert err == pytest.approx(err_ref, rel=1e-12)


def test_writer_errors(ds):
    x = np.zeros((10, 4), np.float32)
    x[3, 1] = np.nan
    snap = _Snap({0: _Tab(0, x)}, 1)
    with pytest.raises(ds.DataError):
        ds.build_shard_payload(snap, _Plan("full", None, 4), 0)
    with pytest.raises(ds.BoundsError):
        ds.build_shard_payload(_Snap({0: _Tab(0, np.zeros((10, 4), np.float32))}, 1),
                               _Plan("incremental", {0: np.array([10])}, 8), 0)


# --- restore ------------------------------------------------------------------------

@pytest.mark.parametrize("bw", (None, 3, 8))
def test_restore_chain_matches_golden(ds, golden, bw):
    g = golden("restore")
    tag = f"bw{bw}"
    rows, d = g[f"{tag}_values_t0"].shape
    chain = []
    for i in range(int(g[f"{tag}_nchain"])):
        chain.append((str(g[f"{tag}_kind{i}"]), [g[f"{tag}_m{i}_s{s}"].tobytes() for s in range(2)]))
    out = ds.restore_chain(chain, {0: (rows, d), 1: (rows, d)}, aux=True)
    for t in range(2):
        assert np.array_equal(u32(out.tables[t].values.cpu().numpy()), u32(g[f"{tag}_values_t{t}"]))
        assert np.array_equal(u32(out.tables[t].aux.cpu().numpy()), u32(g[f"{tag}_aux_t{t}"]))
        assert np.array_equal(out.tracker.since_baseline(t).dirty_rows()[0], g[f"{tag}_base_t{t}"])
    # row-sharded restore: two halves reassemble the same tables
    halves = [ds.restore_chain(chain, {0: (rows, d), 1: (rows, d)}, aux=True,
                               row_range=(lo, hi)) for lo, hi in ((0, 77), (77, rows))]
    for t in range(2):
        cat = np.concatenate([h.tables[t].values.cpu().numpy() for h in halves])
        assert np.array_equal(u32(cat), u32(g[f"{tag}_values_t{t}"]))


@pytest.mark.parametrize("world", (2, 4))
def test_rank_local_restore_chain_vs_oracle(ds, O, world):
    """Row-sharded restore of a 1 full + 3 incremental chain (C5's shape):
    each rank uploads only its rows' records (engine.rank_slices) and its
    tables equal the oracle's restore of the whole chain, rows and
    since-baseline bits; the ranks' uploads add up to the record bytes."""
    from paper_2010_08679_b200.engine import apply_payload
    from paper_2010_08679_b200.sharded import shard_rows
    rng = np.random.default_rng(61)
    rows = {0: 10_000, 1: 333, 2: 70_001}
    vals = {t: rng.standard_normal((r, 16)).astype(np.float32) for t, r in rows.items()}
    chain = [("full", O.build_shard_payload({t: (v, None) for t, v in vals.items()}, "full", None,
                                            8, sorted(rows))[0])]
    for k in range(3):
        sel = {t: np.unique(rng.integers(0, r, r // 3)) for t, r in rows.items()}
        for t in rows:
            vals[t] = vals[t] + np.float32(0.01)
        chain.append(("incremental", O.build_shard_payload(
            {t: (v, None) for t, v in vals.items()}, "incremental", sel, 8, sorted(rows))[0]))
    want = {t: np.zeros((r, 16), np.float32) for t, r in rows.items()}
    bits = {t: np.zeros((r + 7) // 8, np.uint8) for t, r in rows.items()}
    for kind, blob in chain:
        inc = kind == "incremental"
        for tid, sec in O.split_sections(blob, inc):
            O.apply_section(sec, inc, want[tid], None, bits[tid] if inc else None)
    h2d = 0
    for g in range(world):
        lo_hi = {t: shard_rows(r, world, g) for t, r in rows.items()}
        # every table's own rank range: restore_chain takes one range, so do it per table set
        out = {}
        for t, (lo, hi) in lo_hi.items():
            part = ds.restore_chain([(k, [b]) for k, b in chain], {t2: (rows[t2], 16) for t2 in rows},
                                    row_range=(lo, hi))
            out[t] = part
        for t, (lo, hi) in lo_hi.items():
            got = out[t].tables[t].values.cpu().numpy()
            assert np.array_equal(u32(got), u32(want[t][lo:hi])), (g, t)
            b_ref = np.unpackbits(bits[t], bitorder="little")[:rows[t]][lo:hi]
            b_got = np.unpackbits(out[t].tracker.baseline_bitmap(t).to_bytes(),
                                  bitorder="little")[:hi - lo]
            assert np.array_equal(b_got, b_ref), (g, t)
    # upload volume of one rank's pass over the chain vs the whole payloads
    tabs = {t: ds.DeviceTable(t, torch.zeros((rows[t] // world + 1, 16), device="cuda"),
                              row_base=0, total_rows=rows[t]) for t in rows}
    for t in tabs:
        tabs[t] = ds.DeviceTable(t, torch.zeros((shard_rows(rows[t], world, 0)[1], 16), device="cuda"),
                                 row_base=0, total_rows=rows[t])
    for kind, blob in chain:
        apply_payload(blob, kind == "incremental", tabs)
        h2d += apply_payload.last_h2d_bytes
    total = sum(len(b) for _, b in chain)
    assert h2d < total * (1.0 / world + 0.05), (h2d, total)


def test_restore_errors(ds, O):
    x = np.random.default_rng(0).normal(size=(4, 5)).astype(np.float32)
    blob, _, _ = O.build_section(0, x, np.array([0, 2]), bitwidth=3)
    shapes = {0: (4, 5)}
    bad = bytearray(blob)
    bad[24 + 16 + 1] |= 0x80
    with pytest.raises(ds.FormatError):
        ds.restore_chain([("incremental", [bytes(bad)])], shapes)
    oob = bytearray(blob)
    oob[24:32] = (4).to_bytes(8, "little")
    with pytest.raises(ds.IntegrityError):
        ds.restore_chain([("incremental", [bytes(oob)])], shapes)
    with pytest.raises(ds.IntegrityError):
        ds.restore_chain([("incremental", [blob])], {1: (4, 5)})
    with pytest.raises(ds.IntegrityError):
        ds.restore_chain([("incremental", [blob])], {0: (4, 6)})
    with pytest.raises(ds.FormatError):
        ds.restore_chain([("incremental", [blob + b"\x01"])], shapes)


# --- packed lookup streams (ds_mark_packed) ---------------------------------------

def test_mark_packed_mixed_widths(ds):
    """Bit-packed and u8 / u16 segments of one stream, every table kind, Zipf
    repeats and ragged lengths: the interval sets equal the unique ids."""
    rng = np.random.default_rng(21)
    rows = {0: 1, 1: 200, 2: 256, 3: 257, 4: 16352, 5: 40_000, 6: 65_536, 7: 65_537, 8: 12_000_000,
            9: 20_000_000}
    look = {}
    for t, r in rows.items():
        n = int(rng.integers(0, 30_000))
        hot = rng.integers(0, r, 4)
        look[t] = np.where(rng.random(n) < 0.6, hot[rng.integers(0, 4, n)], rng.integers(0, r, n))
    st = ds.LookupStream.pack(look, rows)
    # bit-packed (4, 12, 20, 24, 28 bits) and plain u8 / u16 segments
    assert [ds.lookup_width(r) for r in rows.values()] == [4, 8, 8, 12, 16, 16, 16, 20, 24, 28]
    assert st.seg_width.tolist() == [4, 8, 8, 12, 16, 16, 16, 20, 24, 28]
    tr = ds.ModelTracker(rows)
    tr.mark_packed(st.to(tr.device))
    view = tr.capture()
    for t in rows:
        assert np.array_equal(view.interval_rows[t], np.unique(look[t])), t


def test_mark_packed_bounds(ds):
    """Packed widths cannot hold out-of-range ids: LookupStream.pack rejects
    them on the host (BoundsError, nothing marked); the kernel-side bounds
    flag of 32/64-bit streams is covered by test_mark_batch_table_kinds_and_bounds."""
    rows = {0: 100, 1: 70_000}
    for bad in ({0: np.array([5, 100])}, {1: np.array([1, 70_000])}, {1: np.array([-3])}):
        with pytest.raises(ds.BoundsError):
            ds.LookupStream.pack(bad, rows)
    tr = ds.ModelTracker(rows)
    st = ds.LookupStream.pack({0: np.array([5, 99]), 1: np.array([1, 69_999, 1])}, rows)
    tr.mark_packed(st.to(tr.device))
    view = tr.capture()
    assert view.interval_rows[0].tolist() == [5, 99]
    assert view.interval_rows[1].tolist() == [1, 69_999]


@pytest.mark.parametrize("scope", ("interval", "since_baseline"))
def test_capture_into_matches_capture(ds, scope):
    """The stall-window form (device ids + counts, fold in the same pass)
    equals capture() + reset_interval (tracker.py:100-124)."""
    rng = np.random.default_rng(8)
    rows = {2: 100_000, 5: 33, 9: 5_000_000, 11: 4096}
    a, b = ds.ModelTracker(rows), ds.ModelTracker(rows)
    for phase in range(3):
        for t, r in rows.items():
            idx = rng.integers(0, r, int(rng.integers(1, 50_000)))
            a.mark(t, idx)
            b.mark(t, idx)
        ids = torch.empty(sum(rows.values()), dtype=torch.int64, device="cuda")
        counts = a.capture_into(ids, None, fold=1, scope=scope)
        view = b.capture()
        b.reset_interval()
        c = counts.cpu().numpy()
        h = ids.cpu().numpy()
        off = 0
        want = view.interval_rows if scope == "interval" else view.baseline_rows
        for k, t in enumerate(sorted(rows)):
            assert np.array_equal(h[off:off + c[k]], want[t]), (phase, t)
            off += c[k]
        assert c[len(rows)] == off


def test_restore_mixed_dims_and_bitwidths_vs_oracle(ds, O):
    """One payload whose sections differ in dim (one restore launch per run of
    equal (dim, bitwidth, aux)); full and incremental; against the oracle's
    apply_section."""
    rng = np.random.default_rng(17)
    shapes = {0: (3000, 16), 1: (500, 8), 2: (2000, 16), 3: (70, 130)}
    vals = {t: rng.standard_normal(sh).astype(np.float32) for t, sh in shapes.items()}
    for kind in ("full", "incremental"):
        for bw in (None, 3, 8):
            sel = {t: np.sort(rng.choice(sh[0], sh[0] // 3, replace=False)) for t, sh in shapes.items()}
            blob, _, _ = O.build_shard_payload({t: (v, None) for t, v in vals.items()}, kind,
                                               sel if kind == "incremental" else None, bw,
                                               sorted(shapes))
            got = ds.restore_chain([(kind, [blob])], shapes)
            for t, (r, dim) in shapes.items():
                want = np.zeros((r, dim), np.float32)
                for tid, sec in O.split_sections(blob, kind == "incremental"):
                    if tid == t:
                        O.apply_section(sec, kind == "incremental", want)
                assert np.array_equal(u32(got.tables[t].values.cpu().numpy()), u32(want)), (kind, bw, t)


# --- payload checksum (store.py:46-47) ---------------------------------------------

@pytest.mark.parametrize("n", (0, 1, 3, 4, 5, 127, 128, 129, 4095, 32767, 32768, 32769, 65536,
                               1_000_003, 20_000_000))
def test_crc32_matches_zlib(ds, n):
    import zlib
    rng = np.random.default_rng(n)
    b = rng.integers(0, 256, n, dtype=np.uint8)
    t = torch.from_numpy(b).cuda()
    assert ds.payload.crc32(t) == zlib.crc32(b.tobytes()) & 0xFFFFFFFF
    if n > 1:  # unaligned start, prefix length
        assert ds.payload.crc32(t[1:], n - 1) == zlib.crc32(b[1:].tobytes()) & 0xFFFFFFFF


def test_crc32_of_a_payload(ds, O):
    import zlib
    rng = np.random.default_rng(3)
    tabs = {t: (rng.standard_normal((2000, 16)).astype(np.float32), None) for t in range(3)}
    blob, _, _ = O.build_shard_payload(tabs, "full", None, 4, [0, 1, 2])
    assert ds.payload.crc32(blob) == zlib.crc32(blob) & 0xFFFFFFFF


# --- training step with tracking folded in (sim.py:140-155) -------------------------

@pytest.mark.parametrize("sorted_runs", (True, False))
def test_apply_batches_matches_np_add_at(ds, sorted_runs):
    """values/aux after several batches equal np.add.at's sequential sums bit
    for bit (repeated rows), and the interval bitmap equals mark()."""
    from paper_2010_08679_b200.train import apply_packed, pack_batches
    rng = np.random.default_rng(12)
    rows, dim = {0: 500, 1: 70_000, 2: 7}, 16
    vals = {t: rng.standard_normal((r, dim)).astype(np.float32) for t, r in rows.items()}
    auxs = {t: rng.random((r, dim)).astype(np.float32) for t, r in rows.items()}
    tabs = {t: ds.DeviceTable(t, torch.from_numpy(vals[t]).cuda(), torch.from_numpy(auxs[t]).cuda())
            for t in rows}
    tr, ref_tr = ds.ModelTracker(rows), ds.ModelTracker(rows)
    batches = []
    for b in range(4):
        batch = {}
        for t, r in rows.items():
            n = int(rng.integers(1, 4096))
            hot = rng.integers(0, r, 5)
            idx = np.where(rng.random(n) < 0.5, hot[rng.integers(0, 5, n)], rng.integers(0, r, n))
            batch[t] = (idx.astype(np.int64), (rng.standard_normal((n, dim)) * 0.01).astype(np.float32))
        batches.append(batch)
    apply_packed(tabs, pack_batches(tabs, batches[:1]), tracker=tr, sorted_runs=sorted_runs)
    apply_packed(tabs, pack_batches(tabs, batches[1:]), tracker=tr, sorted_runs=sorted_runs)
    for batch in batches:
        for t in sorted(batch):
            idx, delta = batch[t]
            np.add.at(vals[t], idx, delta)
            np.add.at(auxs[t], idx, delta * delta)
            ref_tr.mark(t, idx)
    view, ref = tr.capture(), ref_tr.capture()
    for t in rows:
        assert np.array_equal(u32(tabs[t].values.cpu().numpy()), u32(vals[t])), t
        assert np.array_equal(u32(tabs[t].aux.cpu().numpy()), u32(auxs[t])), t
        assert np.array_equal(view.interval_rows[t], ref.interval_rows[t]), t


@pytest.mark.parametrize("n,bits", [(1, 1), (2047, 8), (2049, 9), (100_000, 17), (3_000_001, 29),
                                     (500_000, 32)])
def test_sort_pairs_is_a_stable_sort(ds, n, bits):
    """ds_sort_pairs_u32 (the training step's in-tree radix sort) equals
    numpy's stable argsort on the low key bits, ties in input order."""
    import ctypes
    from paper_2010_08679_b200 import _lib
    rng = np.random.default_rng(n + bits)
    hi = 1 << bits
    keys = rng.integers(0, min(hi, 1 << 31), n, dtype=np.int64)
    keys[rng.random(n) < 0.3] = rng.integers(0, 4) % hi  # heavy ties
    keys = (keys % hi).astype(np.uint32)
    vals = np.arange(n, dtype=np.uint32)
    L = _lib.lib()
    k_in = torch.from_numpy(keys.view(np.int32)).cuda()
    v_in = torch.from_numpy(vals.view(np.int32)).cuda()
    k_out, v_out = torch.empty_like(k_in), torch.empty_like(v_in)
    ws = torch.empty(int(L.ds_sort_workspace_size(n)), dtype=torch.uint8, device="cuda")
    _lib.check(L.ds_sort_pairs_u32(k_in.data_ptr(), v_in.data_ptr(), k_out.data_ptr(), v_out.data_ptr(),
                                   n, bits, ws.data_ptr(), ws.numel(), _lib.stream_handle()), "sort")
    order = np.argsort(keys & np.uint32(hi - 1 if bits < 32 else 0xFFFFFFFF), kind="stable")
    assert np.array_equal(v_out.cpu().numpy().view(np.uint32), vals[order])
    assert np.array_equal(k_out.cpu().numpy().view(np.uint32), keys[order])
    assert np.array_equal(k_in.cpu().numpy().view(np.uint32), keys)  # inputs intact


def test_interval_training_hot_rows_and_bounds(ds):
    """ds_train_apply_interval: a row hit 5,000 times in one interval (runs far
    longer than the 32-occurrence prefetch), singletons, and out-of-range ids
    (BoundsError at the tracker's next sync, never applied)."""
    from paper_2010_08679_b200.train import apply_packed, pack_batches
    rng = np.random.default_rng(77)
    rows, dim = {0: 100_000, 1: 7}, 16
    vals = {t: rng.standard_normal((r, dim)).astype(np.float32) for t, r in rows.items()}
    tabs = {t: ds.DeviceTable(t, torch.from_numpy(vals[t].copy()).cuda()) for t in rows}
    tr = ds.ModelTracker(rows)
    batches = []
    for b in range(3):
        batch = {}
        for t, r in rows.items():
            idx = np.where(rng.random(2000) < 0.85, 3 % r, rng.integers(0, r, 2000)).astype(np.int64)
            batch[t] = (idx, (rng.standard_normal((2000, dim)) * 0.01).astype(np.float32))
        batches.append(batch)
    apply_packed(tabs, pack_batches(tabs, batches), tracker=tr)
    want = {t: vals[t].copy() for t in rows}
    for batch in batches:
        for t in sorted(batch):
            np.add.at(want[t], batch[t][0], batch[t][1])
    for t in rows:
        assert np.array_equal(u32(tabs[t].values.cpu().numpy()), u32(want[t])), t
    bad = [{0: (np.array([5, 100_000, -1, 5]), np.ones((4, dim), np.float32)), 1: batches[0][1]}]
    apply_packed(tabs, pack_batches(tabs, bad), tracker=tr)
    with pytest.raises(ds.BoundsError):
        tr.capture()
    np.add.at(want[0], np.array([5, 5]), np.ones((2, dim), np.float32))
    np.add.at(want[1], bad[0][1][0], bad[0][1][1])
    for t in rows:
        assert np.array_equal(u32(tabs[t].values.cpu().numpy()), u32(want[t])), t


def test_stage_chain_verifies_on_device(ds, golden):
    """Restore-side checksums on the device (store.py:488-507): a good chain
    restores exactly like restore_chain; one flipped byte raises
    IntegrityError before any table is touched."""
    import zlib
    g = golden("restore")
    tag = "bw3"
    rows, d = g[f"{tag}_values_t0"].shape
    chain = [(str(g[f"{tag}_kind{i}"]), [g[f"{tag}_m{i}_s{s}"].tobytes() for s in range(2)])
             for i in range(int(g[f"{tag}_nchain"]))]
    sums = [[zlib.crc32(p) for p in ps] for _, ps in chain]
    shapes = {0: (rows, d), 1: (rows, d)}
    out = ds.restore_chain(ds.stage_chain(chain, sums), shapes, aux=True)
    for t in range(2):
        assert np.array_equal(u32(out.tables[t].values.cpu().numpy()), u32(g[f"{tag}_values_t{t}"]))
    bad = [(k, list(ps)) for k, ps in chain]
    b = bytearray(bad[-1][1][0])
    b[len(b) // 2] ^= 0x40
    bad[-1][1][0] = bytes(b)
    with pytest.raises(ds.IntegrityError):
        ds.stage_chain(bad, sums)


def test_staged_checkpoint_matches_direct(ds, O):
    """Stall-window staging: K3 from the gathered copy on a
    side stream, while the tables are overwritten right after the stall,
    yields the same payload as the direct path (and the oracle)."""
    from paper_2010_08679_b200.sharded import ShardedCheckpointer
    rng = np.random.default_rng(31)
    rows = {0: 300, 1: 70_000, 2: 2_000_000}
    for bw in (8, 4, None):
        vals = {t: rng.standard_normal((r, 16)).astype(np.float32) for t, r in rows.items()}
        tabs = [ds.DeviceTable(t, torch.from_numpy(vals[t]).cuda()) for t in rows]
        look = {t: rng.integers(0, r, 30_000) for t, r in rows.items()}
        ck = ShardedCheckpointer(tabs, bw, device="cuda")
        ck.mark(ds.LookupStream.pack(look, rows).to(tabs[0].values.device))
        stall_end = ck.checkpoint(staged_rows=100_000)
        torch.cuda.current_stream().wait_event(stall_end)
        for t in tabs:  # "training" resumes: the live tables change
            t.values.add_(1.0)
        buf, n = ck.fetch()
        torch.cuda.synchronize()
        sel = {t: np.unique(look[t]) for t in rows}
        ref, _, _ = O.build_shard_payload({t: (vals[t], None) for t in rows}, "incremental", sel, bw,
                                          sorted(rows))
        assert bytes(buf[:n].numpy()) == ref, bw
    # a staging buffer that is too small is reported, not silently truncated
    ck.mark(ds.LookupStream.pack(look, rows).to(tabs[0].values.device))
    ck.checkpoint(staged_rows=1000)
    with pytest.raises(ValueError):
        ck.fetch()


def test_staged_capacity_is_flagged_not_overread(ds):
    """A staging buffer smaller than the dirty total (fresh checkpointer: the
    buffer is exactly staged_rows long) raises at fetch; the writer reads no
    row past the buffer."""
    from paper_2010_08679_b200.sharded import ShardedCheckpointer
    rng = np.random.default_rng(41)
    rows = {0: 2_000_000}
    tabs = [ds.DeviceTable(0, torch.randn((rows[0], 128), device="cuda"))]
    ck = ShardedCheckpointer(tabs, 4, adaptive_overrides={4: None}, device="cuda")
    ck.mark(ds.LookupStream.pack({0: rng.integers(0, rows[0], 200_000)}, rows).to("cuda"))
    ck.checkpoint(staged_rows=64)
    with pytest.raises(ValueError):
        ck.fetch()
    torch.cuda.synchronize()  # the context is healthy: no illegal address
    ck.mark(ds.LookupStream.pack({0: rng.integers(0, rows[0], 1000)}, rows).to("cuda"))
    ck.checkpoint()
    buf, n = ck.fetch()
    assert n == 24 + ck.rec * int(ck.counts[0].item())


@pytest.mark.parametrize("packed", (False, True))
def test_checkpoint_pipeline_payloads(ds, O, packed):
    """CheckpointPipeline (the e2e path): 5 consecutive checkpoints through
    the double-buffered H2D -> K1/K2/K3 -> D2H slots, each step's D2H'd bytes
    equal to the oracle's payload for that step's lookups (no
    slot aliasing with keep_outputs)."""
    from paper_2010_08679_b200.pipeline import CheckpointPipeline
    from paper_2010_08679_b200.sharded import ShardedCheckpointer
    rng = np.random.default_rng(51)
    rows = {0: 5000, 1: 300_000, 2: 40}
    vals = {t: rng.standard_normal((r, 16)).astype(np.float32) for t, r in rows.items()}
    tabs = [ds.DeviceTable(t, torch.from_numpy(vals[t]).cuda()) for t in rows]
    ck = ShardedCheckpointer(tabs, 8, device="cuda")
    steps = [{t: rng.integers(0, r, int(rng.integers(1, 20_000))) for t, r in rows.items()}
             for _ in range(5)]
    cap = max(sum(v.size for v in st.values()) for st in steps)
    pipe = CheckpointPipeline(ck, cap * 8, torch.uint8 if packed else torch.int32,
                              keep_outputs=True)
    for st in steps:
        if packed:
            pipe.submit(ds.LookupStream.pack(st, rows))
        else:
            idx = torch.from_numpy(np.concatenate([st[t] for t in rows]).astype(np.int32))
            seg = np.concatenate([[0], np.cumsum([st[t].size for t in rows])]).astype(np.int64)
            pipe.submit(idx.pin_memory(), seg, np.array(list(rows), np.int64))
    outs = pipe.drain()
    assert len(outs) == len(steps)
    for st, got in zip(steps, outs):
        sel = {t: np.unique(st[t]) for t in rows}
        want, _, _ = O.build_shard_payload({t: (vals[t], None) for t in rows}, "incremental", sel,
                                           8, sorted(rows))
        assert got == want


@pytest.mark.parametrize("bw", (8, 4))
def test_checkpoints_overlapped_with_training(ds, O, bw):
    """TrainingCheckpointLoop (north star item 4): interval k's payload is
    written from the staged copy and copied out while interval k+1's
    training steps (ds_train_apply, np.add.at semantics, dirty bits marked
    on the fly) already mutate the tables; every payload still equals the
    oracle's for the tables as they were at the end of interval k."""
    from paper_2010_08679_b200.pipeline import TrainingCheckpointLoop
    from paper_2010_08679_b200.sharded import ShardedCheckpointer
    from paper_2010_08679_b200.train import apply_packed, pack_batches
    rng = np.random.default_rng(71)
    rows = {0: 3000, 1: 200_000, 2: 50}
    dim = 16
    tabs = {t: ds.DeviceTable(t, torch.from_numpy(rng.standard_normal((r, dim)).astype(np.float32)).cuda())
            for t, r in rows.items()}
    ck = ShardedCheckpointer([tabs[t] for t in sorted(rows)], bw, adaptive_overrides={bw: None},
                             device="cuda")
    loop = TrainingCheckpointLoop(ck, staged_rows=sum(rows.values()))
    want = []
    for k in range(4):
        touched = {t: [] for t in rows}
        for b in range(6):  # the interval's training steps
            batch = {}
            for t, r in rows.items():
                idx = rng.integers(0, r, int(rng.integers(1, 1500)))
                batch[t] = (idx, (rng.standard_normal((idx.size, dim)) * 0.01).astype(np.float32))
                touched[t].append(idx)
            apply_packed(tabs, pack_batches(tabs, [batch]), tracker=ck.tracker, sorted_runs=False)
        stall_end = loop.checkpoint()
        # the tables as the checkpoint saw them (test-only sync at the stall's end)
        stall_end.synchronize()
        snap = {t: (tabs[t].values.cpu().numpy(), None) for t in rows}
        sel = {t: np.unique(np.concatenate(touched[t])) for t in rows}
        want.append(O.build_shard_payload(snap, "incremental", sel, bw, sorted(rows),
                                          adaptive={bw: (1, 0.5)})[0])
    got = loop.drain()
    loop.close()
    assert len(got) == len(want)
    for g, w in zip(got, want):
        assert g == w


def test_empty_inputs(ds, O):
    """Empty marks, empty selections, zero-row codec calls, header-only
    payloads and empty lookup streams behave like the reference."""
    bm = ds.DirtyBitmap(0, 100)
    bm.mark(np.zeros(0, np.int64))
    ids, frac = bm.dirty_rows()
    assert ids.size == 0 and frac == 0.0 and bm.popcount() == 0
    tr = ds.ModelTracker({0: 1, 1: 50})
    view = tr.capture()
    assert all(view.interval_rows[t].size == 0 for t in (0, 1))
    x = np.zeros((0, 16), np.float32)
    lo = hi = np.zeros(0, np.float32)
    assert ds.quantize_rows(x, lo, hi, 4).shape == (0, 16)
    assert ds.pack_code_rows(np.zeros((0, 16), np.uint8), 4).shape[0] == 0
    # header-only payload: every table selected with no rows
    tabs = {t: (np.ones((10, 16), np.float32), None) for t in range(3)}
    sel = {t: np.zeros(0, np.int64) for t in range(3)}

    class _T:
        def __init__(self, t):
            self.table_id, self.values, self.aux = t, tabs[t][0], None

    class _S:
        def shard_tables(self, sid):
            return [_T(t) for t in range(3)]

    class _P:
        kind, rows, bitwidth = "incremental", sel, 8

    blob, q, err = ds.build_shard_payload(_S(), _P(), 0)
    ref, q_ref, err_ref = O.build_shard_payload(tabs, "incremental", sel, 8, [0, 1, 2])
    assert blob == ref and q == q_ref == 0 and err == err_ref == 0.0
    out = ds.restore_chain([("incremental", [blob])], {t: (10, 16) for t in range(3)})
    assert all(float(out.tables[t].values.abs().sum()) == 0.0 for t in range(3))
    # an empty lookup stream and a checkpoint with nothing dirty
    from paper_2010_08679_b200.sharded import ShardedCheckpointer
    rows = {0: 10, 1: 100_000}
    st = ds.LookupStream.pack({0: np.zeros(0, np.int64), 1: np.zeros(0, np.int64)}, rows)
    dt = [ds.DeviceTable(t, torch.ones((r, 16), device="cuda")) for t, r in rows.items()]
    ck = ShardedCheckpointer(dt, 8, device="cuda")
    ck.step(st.to(dt[0].values.device))
    buf, n = ck.fetch()
    torch.cuda.synchronize()
    assert n == 2 * 24  # two headers, no records


def test_mark_batch_unaligned_segments(ds):
    """Segments that do not start on 16 bytes take the grid-stride K1 form."""
    rng = np.random.default_rng(23)
    rows = {0: 1000, 1: 300_000, 2: 7}
    tr = ds.ModelTracker(rows)
    idx, seg = [], [0]
    for t, r in rows.items():
        a = rng.integers(0, r, int(rng.integers(1, 3000)) * 2 + 1)  # odd lengths
        idx.append(a)
        seg.append(seg[-1] + a.size)
    for dtype in (torch.int32, torch.int64):
        tr.mark_batch(torch.from_numpy(np.concatenate(idx)).to(dtype).cuda(), np.array(seg),
                      np.array(list(rows)))
        view = tr.capture()
        for k, t in enumerate(rows):
            assert np.array_equal(view.interval_rows[t], np.unique(idx[k])), (dtype, t)
        tr.reset_interval()


@pytest.mark.slow
def test_capture_beyond_32bit_row_counts(ds):
    """Table sets above 2^32 rows take K2's 64-bit-count form (bitmaps only:
    2 x 560 MB)."""
    rows = {0: 3_000_000_000, 1: 1_500_000_017}
    tr = ds.ModelTracker(rows)
    marks = {0: np.array([0, 5, 2_999_999_999, 1 << 31, 2_999_999_000]),
             1: np.array([1_500_000_016, 12, 12, 0])}
    for t, m in marks.items():
        tr.mark(t, m)
    view = tr.capture()
    for t, m in marks.items():
        assert np.array_equal(view.interval_rows[t], np.unique(m)), t

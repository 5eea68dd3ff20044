"""Pin the CPU oracle to the reference before trusting it as the checker.

The fixtures in tests/golden/ were produced by importing the reference
`deltasnap` package (tests/golden/make_golden.py).  Every comparison is
bit-exact: codes, dequantized float32 bits, float64 reconstruction errors,
greedy ranges, packed bytes, whole shard payloads and restored tables.
"""

import struct

import numpy as np
import pytest

from oracle import oracle as O

from .conftest import have_reference, import_reference

DIMS = (1, 3, 7, 8, 9, 16, 33, 64, 65, 128, 130)


@pytest.mark.parametrize("d", DIMS)
@pytest.mark.parametrize("n", (2, 3, 4, 8))
def test_codec_matches_reference_golden(golden, d, n):
    g = golden("codec")
    x = g[f"x_d{d}"]
    lo, hi = x.min(axis=1), x.max(axis=1)
    codes = O.quantize_rows(x, lo, hi, n)
    assert np.array_equal(codes, g[f"codes_d{d}_n{n}"])
    deq = O.dequantize_rows(codes, lo, hi, n)
    assert np.array_equal(deq.view(np.uint32), g[f"deq_d{d}_n{n}"].view(np.uint32))
    me = O.reconstruction_errors(x, lo, hi, n)
    assert np.array_equal(me.view(np.uint64), g[f"me_d{d}_n{n}"].view(np.uint64))
    packed = O.pack_code_rows(codes, n)
    assert np.array_equal(packed, g[f"packed_d{d}_n{n}"])
    assert np.array_equal(O.unpack_code_rows(packed, n, d), codes)
    if n != 8:
        amin, amax = O.adaptive_params_rows(x, n, *{2: (25, 0.5), 3: (25, 0.2), 4: (45, 0.2)}[n])
        assert np.array_equal(amin, g[f"amin_d{d}_n{n}"])
        assert np.array_equal(amax, g[f"amax_d{d}_n{n}"])
        assert np.array_equal(O.quantize_rows(x, amin, amax, n), g[f"acodes_d{d}_n{n}"])


@pytest.mark.parametrize("n", (2, 3, 4))
@pytest.mark.parametrize("bins,ratio", [(25, 0.5), (25, 0.2), (45, 0.2), (10, 0.3), (2, 1.0),
                                        (1, 1.0)])
def test_greedy_configs_match_reference_golden(golden, n, bins, ratio):
    g = golden("codec")
    amin, amax = O.adaptive_params_rows(g["cfg_x"], n, bins, ratio)
    assert np.array_equal(amin, g[f"cfg_min_n{n}_b{bins}_r{ratio}"])
    assert np.array_equal(amax, g[f"cfg_max_n{n}_b{bins}_r{ratio}"])


def test_known_answers():
    # tests/test_quant.py:345-346, :103-107, :93-100, :123-135
    assert O.pack_code_rows(np.array([[0, 1, 2, 3]], np.uint8), 2).tobytes() == b"\xe4"
    codes = O.quantize_rows(np.array([[0.5, 1.5, 2.5]], np.float32), np.float32([0.0]),
                            np.float32([3.0]), 2)
    assert codes.tolist() == [[1, 2, 3]]
    x = np.array([[-1.0, 0.0, 2.0]], np.float32)
    assert O.quantize_rows(x, x.min(1), x.max(1), 2).tolist() == [[0, 1, 3]]
    c = np.full((1, 9), 0.123, np.float32)
    q = O.quantize_rows(c, c.min(1), c.max(1), 3)
    assert not q.any()
    assert np.array_equal(O.dequantize_rows(q, c.min(1), c.max(1), 3), c)
    assert O.quantize_rows(np.array([[-5.0, 5.0]], np.float32), np.float32([-1]),
                           np.float32([1]), 4).tolist() == [[0, 15]]
    with pytest.raises(O.OracleError):
        O.unpack_code_rows(np.frombuffer(b"\xc0", np.uint8).reshape(1, 1), 2, 3)
    with pytest.raises(O.OracleError):
        O.pack_code_rows(np.array([[4]], np.uint8), 2)
    # floor(0.49999999999999994 + 0.5) == 1 in IEEE double
    assert O.pairwise_sum([0.49999999999999994, 0.5]) == 1.0


def test_tracker_matches_reference_golden(golden):
    g = golden("tracker")
    rows = [int(r) for r in g["rows"]]
    interval = {t: np.zeros((r + 7) // 8, np.uint8) for t, r in enumerate(rows)}
    baseline = {t: np.zeros((r + 7) // 8, np.uint8) for t, r in enumerate(rows)}
    total = sum(rows)
    for phase in range(3):
        for t, r in enumerate(rows):
            O.mark(interval[t], r, g[f"mark_p{phase}_t{t}"])
        ni = nb = 0
        for t, r in enumerate(rows):
            ids = O.dirty_rows(interval[t], r)
            union = np.zeros_like(interval[t])
            union[:] = interval[t] | baseline[t]
            ids_b = O.dirty_rows(union, r)
            assert np.array_equal(ids, g[f"int_p{phase}_t{t}"])
            assert np.array_equal(ids_b, g[f"base_p{phase}_t{t}"])
            ni += ids.size
            nb += ids_b.size
        assert [ni / total, nb / total] == g[f"frac_p{phase}"].tolist()
        for t in range(len(rows)):
            baseline[t] |= interval[t]
            interval[t][:] = 0


def test_mark_bounds():
    bits = np.zeros(2, np.uint8)
    with pytest.raises(O.OracleError):
        O.mark(bits, 10, [10])
    with pytest.raises(O.OracleError):
        O.mark(bits, 10, [-1])
    assert not bits.any()


@pytest.mark.parametrize("aux", (0, 1))
@pytest.mark.parametrize("bw", (None, 2, 3, 4, 8))
@pytest.mark.parametrize("kind", ("full", "incremental"))
def test_payload_matches_reference_golden(golden, aux, bw, kind):
    g = golden("payload")
    tag = f"aux{aux}"
    tables = {t: (g[f"{tag}_values_t{t}"], g[f"{tag}_aux_t{t}"] if aux else None)
              for t in range(3)}
    rows = {t: g[f"{tag}_rows_t{t}"] for t in range(3)}
    for sid in range(2):
        variants = [(None, "")] + ([({4: (1, 0.5)}, "_naive4")] if bw == 4 else [])
        for ov, suffix in variants:
            key = f"{tag}_bw{bw}_{kind}_s{sid}{suffix}"
            blob, qr, err = O.build_shard_payload(tables, kind, rows, bw,
                                                  [t for t in range(3) if t % 2 == sid],
                                                  chunk_rows=64, adaptive=ov, nthreads=2)
            assert blob == g[key].tobytes(), key
            want_q, want_err = g[key + "_meta"]
            assert qr == want_q
            assert err == want_err  # same chunk order -> bit-identical float


@pytest.mark.parametrize("bw", (None, 3, 8))
def test_restore_chain_matches_reference_golden(golden, bw):
    g = golden("restore")
    tag = f"bw{bw}"
    rows, d = g[f"{tag}_values_t0"].shape
    values = {t: np.zeros((rows, d), np.float32) for t in range(2)}
    aux = {t: np.zeros((rows, d), np.float32) for t in range(2)}
    base = {t: np.zeros((rows + 7) // 8, np.uint8) for t in range(2)}
    for i in range(int(g[f"{tag}_nchain"])):
        inc = str(g[f"{tag}_kind{i}"]) == "incremental"
        for sid in range(2):
            blob = g[f"{tag}_m{i}_s{sid}"].tobytes()
            for tid, sec in O.split_sections(blob, inc):
                O.apply_section(sec, inc, values[tid], aux[tid], base[tid] if inc else None)
    for t in range(2):
        assert np.array_equal(values[t].view(np.uint32), g[f"{tag}_values_t{t}"].view(np.uint32))
        assert np.array_equal(aux[t].view(np.uint32), g[f"{tag}_aux_t{t}"].view(np.uint32))
        assert np.array_equal(O.dirty_rows(base[t], rows), g[f"{tag}_base_t{t}"])


def test_apply_section_rejects_bad_input():
    x = np.random.default_rng(0).normal(size=(4, 5)).astype(np.float32)
    blob, _, _ = O.build_section(0, x, np.array([0, 2]), bitwidth=3)
    dst = np.zeros((4, 5), np.float32)
    bad = bytearray(blob)
    bad[24 + 8 + 8 + 1] |= 0x80  # a padding bit of the first record (15 code bits in 2 bytes)
    with pytest.raises(O.OracleError) as e:
        O.apply_section(bytes(bad), True, dst)
    assert e.value.kind == "FormatError"
    oob = bytearray(blob)
    oob[24:32] = struct.pack("<Q", 4)
    with pytest.raises(O.OracleError) as e:
        O.apply_section(bytes(oob), True, dst)
    assert e.value.kind == "IntegrityError"
    assert not dst.any()


@pytest.mark.skipif(not have_reference(), reason="reference only in the build container")
def test_oracle_matches_live_reference_random_sweep():
    ds = import_reference()
    rng = np.random.default_rng(123)
    for d in (5, 16, 40, 128):
        x = (rng.normal(0, 1, (100, d)) * rng.lognormal(0, 2, (100, 1))).astype(np.float32)
        x[::7, 0] *= 30
        for n in (2, 3, 4):
            cfg = ds.quant.default_adaptive_config(n)
            a = ds.quant.adaptive_params_rows(x, n, cfg)
            b = O.adaptive_params_rows(x, n, cfg.num_bins, cfg.ratio)
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])

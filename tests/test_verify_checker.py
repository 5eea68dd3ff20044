"""The at-scale payload checker (oracle/verify.py) on CPU: it accepts an
oracle-built payload, and flags a flipped id, code byte, param or header."""

import numpy as np
import pytest

from oracle import oracle as O
from oracle.verify import verify_payload


def _case(bitwidth, adaptive, incremental, rng):
    tables = {t: (rng.random((r, 16), dtype=np.float32) * 2 - 1) for t, r in ((0, 3000), (3, 500))}
    ids = {t: np.unique(rng.integers(0, v.shape[0], 700)) for t, v in tables.items()}
    blob = b"".join(O.build_section(t, tables[t], ids[t] if incremental else None,
                                    bitwidth=bitwidth, adaptive=adaptive)[0]
                    for t in sorted(tables))
    exp = [dict(table_id=t, dim=16, ids=ids[t], rows=tables[t].shape[0]) for t in sorted(tables)]
    return np.frombuffer(blob, np.uint8).copy(), exp, (lambda t, r: tables[t][r])


@pytest.mark.parametrize("bitwidth,adaptive", [(8, None), (4, (45, 0.2)), (3, None), (None, None)])
@pytest.mark.parametrize("incremental", (True, False))
def test_checker_accepts_oracle_payload(bitwidth, adaptive, incremental):
    rng = np.random.default_rng(7)
    p, exp, fetch = _case(bitwidth, adaptive, incremental, rng)
    r = verify_payload(p, exp, bitwidth=bitwidth, adaptive=adaptive, incremental=incremental,
                       fetch_rows=fetch, sample=200, nthreads=2)
    assert r["mismatches"] == 0, r
    assert r["headers_checked"] == 2
    assert r["records_checked"] >= 200
    if incremental:
        assert r["ids_checked"] == sum(e["ids"].size for e in exp)


def test_checker_flags_corruption():
    rng = np.random.default_rng(8)
    p, exp, fetch = _case(8, None, True, rng)
    rec = O.record_size(16, 8, False, True)
    kw = dict(bitwidth=8, adaptive=None, incremental=True, fetch_rows=fetch, nthreads=2)
    for off in (24 + 5 * rec, 24 + 5 * rec + 8, 24 + 5 * rec + 20, 4):
        q = p.copy()
        q[off] ^= 0x10
        r = verify_payload(q, exp, sample=10_000, **kw)  # sample >= records: all checked
        assert r["mismatches"] >= 1, off

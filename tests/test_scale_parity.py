"""Parity at the baseline configs' scale (SURVEY 8(c) "large configs: sampled-row
parity"): payloads of hundreds of MB up to past 2^31 bytes written by the
device path (K1 -> K2 -> K3) and checked with oracle/verify.py -- every
header, the whole dirty-id column, >= 1M (or all) strided records, section
ends and every record around byte 2^31, re-derived by the CPU oracle from
the same rows (rows are independent, quant.py:14-15)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ds():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2010_08679_b200 as m
    return m


def _fetch(tables):
    by_id = {t.table_id: t for t in tables}

    def fetch(tid, ids):
        t = by_id[tid]
        idx = torch.from_numpy(np.asarray(ids, np.int64) - t.row_base).cuda()
        return t.values.index_select(0, idx).cpu().numpy()
    return fetch


@pytest.mark.parametrize("bitwidth,adaptive,rows,n_look,sample", [
    (8, None, 6_000_000, 3_000_000, 1_000_000),        # ~2.6M dirty, 370 MB payload
    (4, None, 6_000_000, 3_000_000, 1_000_000),        # the T codec, 210 MB
    (4, (45, 0.2), 2_000_000, 400_000, 200_000),       # reference default 4-bit adaptive
    (2, (25, 0.5), 2_000_000, 400_000, 200_000),       # C4 codec
])
def test_incremental_step_at_scale(ds, bitwidth, adaptive, rows, n_look, sample):
    from oracle.verify import verify_payload
    from paper_2010_08679_b200.sharded import ShardedCheckpointer
    g = torch.Generator(device="cuda")
    g.manual_seed(bitwidth * 100 + rows)
    vals = torch.rand((rows, 128), generator=g, device="cuda").mul_(2).sub_(1)
    # a few constant, tiny-range and huge-range rows among the dirty ones
    vals[7].fill_(0.25)
    vals[11].mul_(1e-30)
    vals[13].mul_(1e30)
    tabs = [ds.DeviceTable(5, vals)]
    look = torch.randint(0, rows, (n_look,), generator=g, device="cuda", dtype=torch.int32)
    look[:3] = torch.tensor([7, 11, 13], dtype=torch.int32)
    overrides = {bitwidth: None} if adaptive is None else {
        bitwidth: ds.AdaptiveConfig(adaptive[0], adaptive[1])}
    ck = ShardedCheckpointer(tabs, bitwidth, adaptive_overrides=overrides, device="cuda")
    look_h = look.cpu().numpy()
    ck.step(ds.LookupStream.pack({5: look_h}, {5: rows}).to("cuda"))
    buf, n = ck.fetch()
    torch.cuda.synchronize()
    exp = [dict(table_id=5, dim=128, ids=np.unique(look_h).astype(np.int64))]
    r = verify_payload(buf[:n].numpy(), exp, bitwidth=bitwidth, adaptive=adaptive,
                       incremental=True, fetch_rows=_fetch(tabs), sample=sample)
    assert r["mismatches"] == 0, r
    assert r["ids_checked"] == exp[0]["ids"].size
    assert r["records_checked"] >= min(sample, exp[0]["ids"].size)
    if adaptive is None:
        assert n >= (256 << 20 if bitwidth == 8 else 160 << 20)


def test_full_checkpoint_past_2_31_bytes(ds):
    """A 2.18 GB full 8-bit section: 64-bit byte offsets in the writer; every
    record around byte 2^31 plus 1M strided records checked."""
    from oracle.verify import verify_payload
    rows = 16_000_000
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    vals = torch.rand((rows, 128), generator=g, device="cuda").mul_(2).sub_(1)
    tabs = [ds.DeviceTable(2, vals)]
    w = ds.ShardWriter(tabs, 8, adaptive=None)
    nbytes = w.payload_bytes(None)
    assert nbytes > (1 << 31)
    payload = torch.empty(nbytes + 16, dtype=torch.uint8, device="cuda")
    w.write(payload)
    total, _ = w.finish()
    assert total == nbytes
    host = payload[:nbytes].cpu().numpy()
    exp = [dict(table_id=2, dim=128, rows=rows)]
    r = verify_payload(host, exp, bitwidth=8, adaptive=None, incremental=False,
                       fetch_rows=_fetch(tabs), sample=1_000_000)
    assert r["mismatches"] == 0, r
    assert r["records_past_2^31_checked"] > 4096

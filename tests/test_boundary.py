"""CPU-side checks of the drop-in boundary: the C-ABI library loads and exports
every symbol include/deltasnap_cuda.h declares; host logic (headers, layout)
behaves like the reference.  No kernel is launched here."""

import ctypes
import os
import re
import struct

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "deltasnap_cuda.h")
LIB = os.path.join(ROOT, "paper_2010_08679_b200", "libdeltasnap_cuda.so")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^DS_API [^(]*?\b(ds_\w+)\(", text, flags=re.M)))


def test_header_declares_the_abi():
    syms = declared_symbols()
    for s in ("ds_mark", "ds_capture", "ds_write_payload", "ds_restore_section",
              "ds_quantize_rows", "ds_adaptive_params_rows", "ds_pack_code_rows"):
        assert s in syms


@pytest.mark.skipif(not os.path.exists(LIB), reason="build() first")
def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(LIB)
    for s in declared_symbols():
        assert hasattr(lib, s), s
    lib.ds_version.restype = ctypes.c_char_p
    assert b"sm_100a" in lib.ds_version()
    lib.ds_record_size.restype = ctypes.c_int64
    lib.ds_record_size.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int]
    # payload.py:68-76 record sizes: mode 1 dim 7 4-bit = 12 (+8 incremental), fp32 + aux
    assert lib.ds_record_size(7, 4, 0, 0) == 12
    assert lib.ds_record_size(7, 4, 0, 1) == 20
    assert lib.ds_record_size(3, 0, 1, 0) == 24


@pytest.mark.skipif(not os.path.exists(LIB), reason="build() first")
def test_python_binding_signatures_cover_the_header():
    from paper_2010_08679_b200 import _lib
    assert set(declared_symbols()) == set(_lib._SIGNATURES)
    _lib.lib()


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2010_08679_b200")
    for name in os.listdir(pkg):
        if name.endswith(".py"):
            src = open(os.path.join(pkg, name)).read()
            assert "oracle" not in re.sub(r"#.*", "", src).replace('"""', ""), name


def test_parse_headers_validation():
    from paper_2010_08679_b200 import FormatError
    from paper_2010_08679_b200.payload import (HEADER_SIZE, pack_header, parse_headers,
                                               parse_shard_payload, record_size)
    assert HEADER_SIZE == 24
    h = pack_header(7, 0, 2, None, 0, False)
    assert h[:4] == b"CNR1" and h[20] == 32 and h[21] == 0
    assert parse_headers(b"", False) == []
    sec = pack_header(3, 2, 5, 3, 1, False) + bytes(2 * record_size(5, 1, 3, False, True))
    infos = parse_headers(sec, True)
    assert infos[0].rows == 2 and infos[0].record_size == 8 + 8 + 2
    for cut in range(1, len(sec)):
        with pytest.raises(FormatError):
            parse_headers(sec[:cut], True)
    with pytest.raises(FormatError):
        parse_headers(sec + b"\x00", True)
    bad = bytearray(sec)
    bad[23] = 1
    with pytest.raises(FormatError):
        parse_headers(bytes(bad), True)
    bad = bytearray(sec)
    bad[20] = 5
    with pytest.raises(FormatError):
        parse_headers(bytes(bad), True)
    bad = bytearray(sec)
    bad[21] = 2
    with pytest.raises(FormatError):
        parse_headers(bytes(bad), True)
    bad = bytearray(sec)
    bad[:4] = b"XXXX"
    with pytest.raises(FormatError):
        parse_headers(bytes(bad), True)
    secs = parse_shard_payload(sec, True)
    assert secs[0].row_indices.tolist() == [0, 0] and secs[0].codes.shape == (2, 2)


def test_serialize_section_matches_oracle_layout():
    from oracle import oracle as O
    from paper_2010_08679_b200.payload import TableSection, parse_shard_payload, serialize_section
    rng = np.random.default_rng(0)
    x = rng.normal(size=(6, 9)).astype(np.float32)
    sel = np.array([0, 2, 3, 5], np.int64)
    for bw in (2, 3, 4, 8):
        blob, _, _ = O.build_section(4, x, sel, bitwidth=bw)
        back = parse_shard_payload(blob, True)[0]
        assert back.row_indices.tolist() == sel.tolist()
        assert serialize_section(back, True) == blob
        lo, hi = O.row_minmax(x[sel])
        assert np.array_equal(back.params[:, 0], lo) and np.array_equal(back.params[:, 1], hi)
    sec = TableSection(table_id=1, dim=9, mode=0, values=x)
    assert serialize_section(sec, False) == O.build_section(1, x, None, bitwidth=None)[0]
    assert struct.unpack_from("<Q", serialize_section(sec, False), 8)[0] == 6


def test_pack_ids_bitstream():
    """LookupStream wire format: ids LSB-first at `bits` bits (ds_mark_packed)."""
    import numpy as np
    from paper_2010_08679_b200.tracker import lookup_width, pack_ids
    rng = np.random.default_rng(4)
    for bits in (1, 3, 7, 8, 9, 13, 16, 17, 24, 31):
        a = rng.integers(0, 1 << bits, 1000 + bits)
        p = pack_ids(a, bits)
        assert p.size == (a.size * bits + 7) // 8
        stream = int.from_bytes(p.tobytes(), "little")
        got = [(stream >> (i * bits)) & ((1 << bits) - 1) for i in range(a.size)]
        assert got == a.tolist(), bits
    assert [lookup_width(r) for r in (1, 2, 3, 256, 257, 1 << 28, (1 << 28) + 1, 1 << 31,
                                      (1 << 31) + 1)] == [4, 4, 4, 8, 12, 28, 32, 32, 64]


def test_ctypes_structs_match_the_header_layout(tmp_path):
    """Every struct the Python binding passes through the C ABI has the
    header's size and field offsets (gcc compiles a probe against the header)."""
    import shutil
    import subprocess
    from paper_2010_08679_b200 import _lib
    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    mirrors = {"ds_table_desc": _lib.TableDesc, "ds_ckpt_params": _lib.CkptParams,
               "ds_restore_sec": _lib.RestoreSec, "ds_train_table": _lib.TrainTable,
               "ds_peer_exchange": _lib.PeerExchange}
    lines = ['#include <stdio.h>', '#include <stddef.h>', f'#include "{HEADER}"', "int main(void) {"]
    for c, py in mirrors.items():
        t = c if c != "ds_peer_exchange" else "struct ds_peer_exchange"
        lines.append(f'printf("{c} size %zu\\n", sizeof({t}));')
        for f, _ in py._fields_:
            lines.append(f'printf("{c} {f} %zu\\n", offsetof({t}, {f}));')
    lines += ["return 0;", "}"]
    src = tmp_path / "probe.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "probe"
    subprocess.run(["gcc", "-o", str(exe), str(src)], check=True)
    got = dict(l.rsplit(" ", 1) for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                          check=True).stdout.splitlines())
    for c, py in mirrors.items():
        assert int(got[f"{c} size"]) == ctypes.sizeof(py), c
        for f, _ in py._fields_:
            assert int(got[f"{c} {f}"]) == getattr(py, f).offset, (c, f)

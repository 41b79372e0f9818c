"""BTSR containers (tensor_io.hpp:14-37, tensor_io.cpp): the Python writer is byte-identical to
the reference writer, the header checks give the reference's IoError texts (CPU), and the
device loader / GPU pack flows match the reference reader and pack (GPU). The reference runs
from oracle/_ref (its own sources, compiled unmodified)."""
import os
import struct

import numpy as np
import pytest

from paper_2306_08960_b200 import api, btsr, data


def _rand_bits(rng, rows, cols, lane=512):
    w, wpr = data.random_words(rng, rows, cols, lane)
    return api.BitMatrix.from_words(rows, cols, wpr, w)


def _rand_csr(rng, rows, cols, dens=0.1):
    mask = rng.random((rows, cols)) < dens
    r, c = np.nonzero(mask)
    rp = np.zeros(rows + 1, np.uint64)
    np.add.at(rp, r + 1, 1)
    rp = np.cumsum(rp).astype(np.uint64)
    return api.CsrMatrix.create(rows, cols, rp, c.astype(np.uint64),
                                rng.uniform(-1, 1, c.size).astype(np.float32))


def _bytes(path):
    with open(path, "rb") as f:
        return f.read()


def test_writer_matches_reference(ref, tmp_path):
    rng = np.random.default_rng(1)
    for rows, cols in [(0, 5), (3, 1), (17, 700), (64, 64)]:
        a = rng.standard_normal((rows, cols)).astype(np.float32)
        btsr.store_tensor(str(tmp_path / "ours.d"), a)
        ref.store_dense(str(tmp_path / "ref.d"), a)
        assert _bytes(tmp_path / "ours.d") == _bytes(tmp_path / "ref.d")
        b = _rand_bits(rng, rows, cols, 64 if cols < 100 else 512)
        btsr.store_tensor(str(tmp_path / "ours.b"), b)
        ref.store_bit(str(tmp_path / "ref.b"), b.words, rows, cols)
        assert _bytes(tmp_path / "ours.b") == _bytes(tmp_path / "ref.b")
        c = _rand_csr(rng, rows, cols)
        btsr.store_tensor(str(tmp_path / "ours.c"), c)
        ref.store_csr(str(tmp_path / "ref.c"), rows, cols, c.row_ptr, c.col_idx, c.vals)
        assert _bytes(tmp_path / "ours.c") == _bytes(tmp_path / "ref.c")
    t, h, m, wpr = data.random_planes(rng, 9, 130)
    for s, g in [(0.5, None), (np.float32(0.1), np.float32(1.25))]:
        bm = lambda w: api.BitMatrix.from_words(9, 130, wpr, w)  # noqa: E731
        btsr.store_thm_planes(str(tmp_path / "ours"), api.ThmPlanes(bm(t), bm(h), bm(m), float(s),
                                                                    None if g is None else float(g)))
        ref.store_thm_planes(str(tmp_path / "ref"), t, h, m, 130, float(s), None if g is None else float(g))
        for suffix in (".t.btsr", ".h.btsr", ".m.btsr", ".json"):
            assert _bytes(str(tmp_path / "ours") + suffix) == _bytes(str(tmp_path / "ref") + suffix), suffix


def _corrupt_headers(tmp_path):
    """(name, bytes) of files whose defect the header / size checks catch."""
    ok_bit = b"BTSR" + struct.pack("<IBQQ", 1, 1, 2, 64) + struct.pack("<Q", 1) + b"\0" * 16
    return [
        ("magic", b"BTSX" + ok_bit[4:]),
        ("version", b"BTSR" + struct.pack("<IBQQ", 2, 1, 2, 64)),
        ("kind", b"BTSR" + struct.pack("<IBQQ", 1, 7, 2, 64)),
        ("short_header", b"BTSR\x01\x00"),
        ("overflow", b"BTSR" + struct.pack("<IBQQ", 1, 0, 1 << 30, 1 << 30)),
        ("truncated", ok_bit[:-3]),
        ("trailing", ok_bit + b"\0"),
        ("empty", b""),
    ]


def test_header_errors_match_reference(ref, tmp_path):
    from paper_2306_08960_b200 import _lib
    for name, blob in _corrupt_headers(tmp_path):
        path = str(tmp_path / f"{name}.btsr")
        with open(path, "wb") as f:
            f.write(blob)
        rc_ref, msg_ref = ref.load_check(path)
        assert rc_ref == 5, name
        with pytest.raises(api.IoError) as e:
            btsr.read_header(path)
        assert str(e.value) == msg_ref, name
    with pytest.raises(api.IoError) as e:
        btsr.read_header(str(tmp_path / "missing.btsr"))
    assert str(e.value) == ref.load_check(str(tmp_path / "missing.btsr"))[1]
    assert _lib.ERR_IO == 5


# ------------------------------------------------------------------ GPU
def _payload_corruptions(rng, tmp_path):
    """(name, path, kind) of files whose defect only the payload / object checks catch."""
    out = []
    def write(name, blob, kind=-1):
        p = str(tmp_path / f"{name}.btsr")
        with open(p, "wb") as f:
            f.write(blob)
        out.append((name, p, kind))
    hdr = lambda k, r, c: b"BTSR" + struct.pack("<IBQQ", 1, k, r, c)  # noqa: E731
    write("padding", hdr(1, 2, 65) + struct.pack("<Q", 2) + struct.pack("<4Q", 0, 0, 0, 4))
    write("padding_word", hdr(1, 1, 64) + struct.pack("<Q", 2) + struct.pack("<2Q", 7, 1))
    write("wpr_small", hdr(1, 1, 130) + struct.pack("<Q", 2) + struct.pack("<2Q", 0, 0))
    write("dense_nan", hdr(0, 1, 3) + struct.pack("<3f", 1.0, float("nan"), 2.0))
    csr = lambda r, c, rp, ci, v: (hdr(2, r, c) + struct.pack("<Q", len(ci)) +  # noqa: E731
                                   struct.pack(f"<{len(rp)}Q", *rp) + struct.pack(f"<{len(ci)}Q", *ci) +
                                   struct.pack(f"<{len(v)}f", *v))
    write("csr_start", csr(2, 4, [1, 1, 1], [2], [1.0]))
    write("csr_monotone", csr(2, 4, [0, 2, 1], [0], [1.0]))
    write("csr_nnz", csr(2, 4, [0, 1, 2], [0], [1.0]))
    write("csr_range", csr(2, 4, [0, 1, 2], [0, 4], [1.0, 2.0]))
    write("csr_increasing", csr(2, 4, [0, 2, 2], [3, 3], [1.0, 2.0]))
    write("csr_nan", csr(1, 4, [0, 1], [1], [float("inf")]))
    write("kind_mismatch", hdr(0, 1, 1) + struct.pack("<f", 1.0), kind=1)
    return out


@pytest.mark.gpu
def test_device_load_roundtrip(tmp_path):
    rng = np.random.default_rng(2)
    a = rng.standard_normal((33, 70)).astype(np.float32)
    b = _rand_bits(rng, 129, 1000)
    c = _rand_csr(rng, 40, 300, 0.05)
    for name, obj in (("d", a), ("b", b), ("c", c)):
        btsr.store_tensor(str(tmp_path / name), obj)
    d = btsr.load_dev(str(tmp_path / "d"), "dense")
    assert np.array_equal(d["data"].cpu().numpy(), a)
    w = btsr.load_dev(str(tmp_path / "b"))
    assert w["kind"] == "bit" and w["words_per_row"] == b.words_per_row()
    assert np.array_equal(w["data"].cpu().numpy().view(np.uint64), b.words)
    s = btsr.load_dev(str(tmp_path / "c"), "csr")
    assert np.array_equal(s["row_ptr"].cpu().numpy().view(np.uint64), c.row_ptr)
    assert np.array_equal(s["col_idx"].cpu().numpy().view(np.uint64), c.col_idx)
    assert np.array_equal(s["vals"].cpu().numpy(), c.vals)
    # larger than one pinned chunk (8 MiB): 4096 x 4096 signs = 2 MiB words, 64 MiB dense
    big = rng.standard_normal((4096, 4096)).astype(np.float32)
    btsr.store_tensor(str(tmp_path / "big"), big)
    assert np.array_equal(btsr.load_dev(str(tmp_path / "big"))["data"].cpu().numpy(), big)


@pytest.mark.gpu
def test_device_load_errors_match_reference(ref, tmp_path):
    rng = np.random.default_rng(3)
    for name, path, kind in _payload_corruptions(rng, tmp_path):
        rc_ref, msg_ref = ref.load_check(path, kind)
        assert rc_ref == 5, (name, msg_ref)
        want = None if kind < 0 else ("dense", "bit", "csr")[kind]
        with pytest.raises(api.IoError) as e:
            btsr.load_dev(path, want)
        assert str(e.value) == msg_ref, name


@pytest.mark.gpu
def test_thm_planes_load_and_validation_match_reference(ref, tmp_path):
    rng = np.random.default_rng(4)
    t, h, m, wpr = data.random_planes(rng, 20, 300)
    pre = str(tmp_path / "p")
    ref.store_thm_planes(pre, t, h, m, 300, 0.25, 2.0)
    got = btsr.load_thm_planes_dev(pre)
    assert got["scale"] == 0.25 and got["gamma"] == 2.0
    assert np.array_equal(got["t"].cpu().numpy().view(np.uint64), t)
    # illegal planes: t and h both set (written with the Python writer, read by both readers)
    for bad, pos in (("th", (5, 1)), ("tm", (7, 2))):
        tt, hh, mm = t.copy(), h.copy(), m.copy()
        r, wi = pos
        if bad == "th":
            tt[r, wi] |= 1
            hh[r, wi] |= 1
            mm[r, wi] |= 1
        else:
            tt[r, wi] |= 2
            mm[r, wi] &= ~np.uint64(2)
            hh[r, wi] &= ~np.uint64(2)
        bm = lambda w: api.BitMatrix.from_words(20, 300, wpr, w)  # noqa: E731
        p2 = str(tmp_path / bad)
        for name, w in (("t", tt), ("h", hh), ("m", mm)):
            btsr.store_tensor(f"{p2}.{name}.btsr", bm(w))
        with open(p2 + ".json", "w") as f:
            f.write('{"gamma": null, "s": 1.0}\n')
        rc_ref, msg_ref = ref.load_check(p2, 3)
        assert rc_ref == 5
        with pytest.raises(api.IoError) as e:
            btsr.load_thm_planes_dev(p2)
        assert str(e.value) == msg_ref


@pytest.mark.gpu
def test_cli_pack_matches_reference_pack(ref, tmp_path):
    from paper_2306_08960_b200 import cli
    rng = np.random.default_rng(5)
    a = rng.standard_normal((70, 1000)).astype(np.float32)
    a[0, :5] = 0.0
    src = str(tmp_path / "w.btsr")
    btsr.store_tensor(src, a)
    assert cli.main(["pack", "--input", src, "--output", str(tmp_path / "ours.bits"), "--mode", "sign"]) == 0
    words, wpr = ref.pack_signs(a)
    ref.store_bit(str(tmp_path / "ref.bits"), words, 70, 1000)
    assert _bytes(tmp_path / "ours.bits") == _bytes(tmp_path / "ref.bits")
    x = (rng.integers(-2, 9, (70, 1000)) * 0.25).astype(np.float32)  # includes .5 ties
    btsr.store_tensor(src, x)
    assert cli.main(["pack", "--input", src, "--output", str(tmp_path / "ours"), "--mode", "thm",
                     "--step", "0.5"]) == 0
    lv = ref.quantize_2bit(x, 0.5)
    t, h, m, _ = ref.decompose_thm(lv, 0.5)
    ref.store_thm_planes(str(tmp_path / "ref"), t, h, m, 1000, 0.5)
    for suffix in (".t.btsr", ".h.btsr", ".m.btsr", ".json"):
        assert _bytes(str(tmp_path / "ours") + suffix) == _bytes(str(tmp_path / "ref") + suffix), suffix
    assert cli.main(["pack", "--input", str(tmp_path / "nope.btsr"), "--output", "x"]) == 3


@pytest.mark.gpu
def test_cli_pack_apb_matches_reference(ref, tmp_path):
    """`pack --mode apb` (bitmm_main.cpp:195-207): init_alpha_delta or given parameters,
    apb_forward, decompose_apb on the GPU, store_apb_layer. Every file is byte-identical to the
    reference CLI's."""
    from paper_2306_08960_b200 import cli
    rng = np.random.default_rng(11)
    w = rng.normal(0.0, 0.02, (96, 700)).astype(np.float32)
    w[0, :4] = [0.0, -0.0, 0.5, -0.5]
    src = str(tmp_path / "w.btsr")
    btsr.store_tensor(src, w)
    for params in (None, (0.015, 0.02)):
        extra = [] if params is None else ["--alpha", str(params[0]), "--delta", str(params[1])]
        assert cli.main(["pack", "--input", src, "--output", str(tmp_path / "ours"), "--mode", "apb"]
                        + extra) == 0
        if params is None:
            ref.pack_apb(w, str(tmp_path / "ref"))
        else:
            ref.pack_apb(w, str(tmp_path / "ref"), np.float32(params[0]), np.float32(params[1]))
        for suffix in (".bin.btsr", ".res.btsr", ".json"):
            assert _bytes(str(tmp_path / "ours") + suffix) == _bytes(str(tmp_path / "ref") + suffix), \
                (params, suffix)
    assert cli.main(["pack", "--input", src, "--output", "x", "--mode", "apb", "--alpha", "1"]) == 2


@pytest.mark.gpu
def test_cli_bench_csv(tmp_path):
    from paper_2306_08960_b200 import cli
    out = str(tmp_path / "b.csv")
    assert cli.main(["bench", "--routine", "1x1", "--routine", "2x2", "--routine", "spmm",
                     "--routine", "1x32_ref", "--m", "256", "--k", "512", "--n", "384", "--reps",
                     "3", "--warmup", "1", "--csv", out]) == 0
    lines = open(out).read().splitlines()
    assert lines[0] == "routine,m,k,n,reps,warmup,threads,simd,seconds,gops,gflops,tpp_gops,pct_tpp"
    assert [ln.split(",")[0] for ln in lines[1:]] == ["1x1", "2x2", "spmm", "1x32_ref"]
    assert all(float(ln.split(",")[9]) > 0 for ln in lines[1:])

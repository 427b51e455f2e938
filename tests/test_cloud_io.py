"""Cloud files: the reference's text format and the binary SoA cache."""
import os
import time

import numpy as np
import pytest

import paper_2406_07441_b200 as kf


def _same(a, b):
    assert a.n() == b.n()
    for f in ("x", "y", "kind", "normal_x", "normal_y"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert np.array_equal(a.nbr.offsets, b.nbr.offsets) and np.array_equal(a.nbr.ids, b.nbr.ids)
    for f in ("xpos", "xneg", "ypos", "yneg"):
        assert np.array_equal(getattr(a, f).ids, getattr(b, f).ids), f
    assert np.array_equal(kf.color_points(a).color, kf.color_points(b).color)


def test_binary_cache_roundtrip_matches_text(tmp_path):
    c = kf.generate_naca_ogrid("0012", 96, 24, 12.0)
    kf.save_cloud(c, tmp_path / "c.txt")
    kf.save_cloud(c, tmp_path / "c.bin", binary=True)
    a = kf.load_cloud(tmp_path / "c.txt")
    b = kf.load_cloud(tmp_path / "c.bin")
    _same(c, a)
    _same(c, b)
    la, lb = kf.build_ls_coefficients(a), kf.build_ls_coefficients(b)
    for k in la.split_w:
        assert np.array_equal(la.split_w[k], lb.split_w[k])


def test_binary_cache_rejects_truncated_and_bad_files(tmp_path):
    c = kf.generate_naca_ogrid("0012", 32, 8, 10.0)
    p = tmp_path / "c.bin"
    kf.save_cloud(c, p, binary=True)
    data = p.read_bytes()
    (tmp_path / "t.bin").write_bytes(data[: len(data) // 2])
    with pytest.raises(kf.KinfreeError):
        kf.load_cloud(tmp_path / "t.bin")
    bad = bytearray(data)
    bad[8:16] = (0).to_bytes(8, "little")  # zero points
    (tmp_path / "z.bin").write_bytes(bytes(bad))
    with pytest.raises(kf.KinfreeError):
        kf.load_cloud(tmp_path / "z.bin")
    with pytest.raises(kf.KinfreeError):
        kf.load_cloud(tmp_path / "missing.bin")


def test_binary_cache_loads_faster_than_text(tmp_path):
    c = kf.generate_naca_ogrid("0012", 640, 250, 20.0)  # 160,000 points
    kf.save_cloud(c, tmp_path / "c.txt")
    kf.save_cloud(c, tmp_path / "c.bin", binary=True)
    t0 = time.perf_counter()
    a = kf.load_cloud(tmp_path / "c.txt")
    t1 = time.perf_counter()
    b = kf.load_cloud(tmp_path / "c.bin")
    t2 = time.perf_counter()
    assert a.n() == b.n() == c.n()
    print(f"text {t1 - t0:.3f} s, binary {t2 - t1:.3f} s")
    assert (t2 - t1) < (t1 - t0)


def _variants(tmp_path):
    """Text clouds exercising the parser's edge cases: the reference's own
    save_cloud output, CRLF line ends, comments and blank lines between
    records, no final newline, and one malformed file per error path
    (pointcloud.cpp:301-381)."""
    import paper_2406_07441_b200 as kf
    c = kf.generate_naca_ogrid("0012", 32, 8, 10.0)
    good = tmp_path / "good.txt"
    kf.save_cloud(c, good)
    lines = good.read_text().splitlines()
    out = {"good": "\n".join(lines) + "\n"}
    out["crlf"] = "\r\n".join(lines) + "\r\n"
    out["comments"] = "# cloud\n\n" + lines[0] + "\n" + "\n".join(
        (f"   # c{k}\n\t\n" if k % 37 == 0 else "") + ln for k, ln in enumerate(lines[1:])) + "\n"
    out["nofinalnl"] = "\n".join(lines)
    out["badheader"] = "x\n" + "\n".join(lines[1:])
    out["zeroheader"] = "0\n" + "\n".join(lines[1:])
    out["order"] = "\n".join(lines[:5] + [lines[6], lines[5]] + lines[7:]) + "\n"
    out["kind"] = "\n".join(lines[:9] + [" ".join(["9" if i == 3 else t for i, t in enumerate(lines[9].split())])]
                            + lines[10:]) + "\n"
    out["shortrec"] = "\n".join(lines[:11] + [" ".join(lines[11].split()[:3])] + lines[12:]) + "\n"
    nb = lines[20].split()
    out["missingnbr"] = "\n".join(lines[:20] + [" ".join(nb[:5 + int(nb[4]) - 1])] + lines[21:]) + "\n"
    out["count"] = "\n".join(lines[:-1]) + "\n"
    out["negnn"] = "\n".join(lines[:30] + [" ".join(lines[30].split()[:4] + ["-1"])] + lines[31:]) + "\n"
    out["multi"] = "\n".join(lines[:7] + [lines[8], lines[7]] + lines[9:13] + ["junk"] + lines[14:]) + "\n"
    out["range"] = out["good"].replace(lines[40], " ".join(
        [t if i != 5 else "9999" for i, t in enumerate(lines[40].split())]))
    out["self"] = out["good"].replace(lines[41], " ".join(
        [t if i != 5 else lines[41].split()[0] for i, t in enumerate(lines[41].split())]))
    return out


def test_parallel_text_parser_matches_the_reference_loader(tmp_path):
    """The parallel parser reads exactly what the reference's sequential
    load_cloud reads, and fails on the same line with the same message."""
    import paper_2406_07441_b200 as kf
    from refpy import Reference, ref_available, OracleError
    if not ref_available():
        pytest.skip("reference not built")
    for name, text in _variants(tmp_path).items():
        path = tmp_path / f"{name}.txt"
        path.write_bytes(text.encode())
        try:
            ref = Reference.load(path)
            ref_err = None
        except OracleError as e:
            ref, ref_err = None, str(e)
        try:
            got = kf.load_cloud(path)
            got_err = None
        except kf.KinfreeError as e:
            got, got_err = None, e.reason
        assert (ref_err is None) == (got_err is None), (name, ref_err, got_err)
        if ref_err is not None:
            assert got_err == ref_err, (name, ref_err, got_err)
            continue
        x, y, kind, nx, ny = ref.geometry()
        assert np.array_equal(got.x, x) and np.array_equal(got.y, y) and np.array_equal(got.kind, kind), name
        off, idx = ref.csr(0)
        assert np.array_equal(got.nbr.offsets, off) and np.array_equal(got.nbr.ids, idx), name

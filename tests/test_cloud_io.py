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

"""Host-side ingestion of libkf (CPU only): the generated clouds, split
stencils, LS weights and colours must be the reference's, bit for bit
(north-star item 1), checked against golden hashes produced by the real
reference and, where available, against the live reference build. Cloud file
I/O follows test_pointcloud.cpp's cases.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import paper_2406_07441_b200 as kf
from refpy import Reference, ref_available
from util import hand_cloud, lattice


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def hashes_of(c):
    out = {"n": c.n(), "x": sha(c.x), "y": sha(c.y), "kind": sha(c.kind.astype(np.int32)),
           "nx": sha(c.normal_x), "ny": sha(c.normal_y)}
    for w, name in enumerate(["nbr", "xpos", "xneg", "ypos", "yneg"]):
        L = c._list(w)
        out[name + "_off"] = sha(L.offsets)
        out[name + "_idx"] = sha(L.ids)
    ls = kf.build_ls_coefficients(c)
    out.update(wx=sha(ls.full_wx), wy=sha(ls.full_wy), full_kind=sha(ls.full_kind))
    for name in ["xpos", "xneg", "ypos", "yneg"]:
        out[name + "_w"] = sha(ls.split_w[name])
        out[name + "_one"] = sha(ls.ls_one[name])
        out[name + "_kind"] = sha(ls.split_kind[name])
    out["flagged"] = sha(ls.flagged)
    col = kf.color_points(c)
    out["color"] = sha(col.color)
    out["n_colors"] = col.n_colors
    return out


@pytest.mark.parametrize("name", ["config1", "config2", "small", "odd"])
def test_ingestion_matches_reference_hashes(golden, name):
    with open(os.path.join(golden, "ingest_hashes.json")) as f:
        want = json.load(f)[name]
    spec = want.pop("spec")
    got = hashes_of(kf.generate_naca_ogrid(*spec))
    for k, v in want.items():
        assert got[k] == v, f"{name}: {k} differs from the reference"


def test_generated_counts_and_palette():
    # test_pointcloud.cpp:37-52, test_coloring.cpp:71-77, SURVEY F6
    c = kf.generate_naca_ogrid("0012", 160, 60, 20.0)
    assert c.n() == 9600 and c.count(kf.PointKind.Wall) == 160 and c.count(kf.PointKind.Outer) == 160
    col = kf.color_points(c)
    assert col.n_colors == 4 and np.all(np.bincount(col.color)[1:] == 2400)
    small = kf.generate_naca_ogrid("0012", 32, 8, 10.0)
    deg = np.diff(small.nbr.offsets)
    assert np.all(deg[small.interior_ids] == 8) and np.all(deg[small.wall_ids] == 5)


def test_generator_rejects_bad_input():
    for args in [("00x2", 64, 16, 15.0), ("0012345", 64, 16, 15.0), ("0000", 64, 16, 15.0),
                 ("1012", 64, 16, 15.0), ("0012", 16, 16, 15.0), ("0012", 64, 4, 15.0),
                 ("0012", 64, 16, 5.0)]:
        with pytest.raises(kf.ConfigError):
            kf.generate_naca_ogrid(*args)


def test_cloud_file_round_trip(tmp_path):
    a = kf.generate_naca_ogrid("0012", 40, 10, 11.0)
    path = tmp_path / "cloud.txt"
    kf.save_cloud(a, path)
    b = kf.load_cloud(path)
    assert b.n() == a.n()
    for attr in ["x", "y", "kind", "normal_x", "normal_y"]:
        assert np.array_equal(getattr(a, attr), getattr(b, attr))
    assert np.array_equal(a.nbr.offsets, b.nbr.offsets) and np.array_equal(a.nbr.ids, b.nbr.ids)
    assert hashes_of(a) == hashes_of(b)


def test_cloud_file_toy_and_errors(tmp_path):
    toy = tmp_path / "toy.txt"
    toy.write_text("# toy strip\n5\n1 0 0 0 3 2 3 4 0 -1\n2 0 1 1 3 1 3 5\n3 1 0.5 1 4 1 2 4 5\n"
                   "4 0 2 1 3 1 3 5\n5 1 2.5 2 3 2 3 4 0.37139067635410372 0.92847669088525941\n")
    c = kf.load_cloud(toy)
    assert (c.count(kf.PointKind.Wall), c.count(kf.PointKind.Interior), c.count(kf.PointKind.Outer)) == (1, 3, 1)
    bad = tmp_path / "bad.txt"
    bad.write_text("4\n1 0 0 1 3 2 3 4\n2 1 0 1 2 1 3\n3 0 1 1 3 1 2 4\n4 1 1 1 3 1 2 3\n")
    with pytest.raises(kf.KinfreeError, match="point 2"):
        kf.load_cloud(bad)
    parse = tmp_path / "parse.txt"
    parse.write_text("2\n1 0 0 1 3 2 2 2\n2 oops 0 1 3 1 1 1\n")
    with pytest.raises(kf.KinfreeError, match=":3:"):
        kf.load_cloud(parse)
    with pytest.raises(kf.KinfreeError, match="cannot open"):
        kf.load_cloud(tmp_path / "missing.txt")


def test_split_stencil_partition_and_ties():
    # test_pointcloud.cpp:70-110
    c = kf.PointCloud.from_arrays(*hand_cloud([(0, 0), (-1, 0.2), (-0.5, -0.1), (1, 0.3), (2, -0.2)],
                                              [[1, 2, 3, 4], [0], [0], [0], [0]]))
    assert list(c.xneg[0]) == [1, 2] and list(c.xpos[0]) == [3, 4]
    t = kf.PointCloud.from_arrays(*hand_cloud([(0, 0), (0, 1), (1, 0), (-1, -1)],
                                              [[1, 2, 3], [0], [0], [0]]))
    assert 1 in list(t.xpos[0]) and 1 in list(t.xneg[0])
    s = kf.PointCloud.from_arrays(*hand_cloud([(0, 0), (1, 1), (2, 2), (-1, -1)],
                                              [[1, 2, 3], [0], [0], [0]]))
    assert 0 in list(s.stencil_report.singular_points)


def test_set_colors_validates():
    pts, nbrs = lattice(4, 4)
    c = kf.PointCloud.from_arrays(*hand_cloud(pts, nbrs))
    with pytest.raises(kf.ConfigError):
        kf.set_colors(c, np.ones(16, np.int32))
    good = kf.color_points(c).color
    kf.set_colors(c, good)


@pytest.mark.skipif(not ref_available(), reason="reference build (oracle/_ref) not present")
def test_ingestion_matches_live_reference_on_arbitrary_clouds(tmp_path):
    rng = np.random.default_rng(314)
    for trial in range(5):
        n = 60 + trial
        pts = rng.uniform(0, 1, (n, 2))
        nbrs = []
        for i in range(n):
            k = rng.integers(3, 8)
            cand = [q for q in rng.permutation(n) if q != i][:k]
            nbrs.append(cand)
        arrs = hand_cloud([tuple(p) for p in pts], nbrs)
        c = kf.PointCloud.from_arrays(*arrs)
        r = Reference.from_arrays(*arrs)
        for w in range(5):
            a, b = c._list(w), r.csr(w)
            assert np.array_equal(a.offsets, b[0]) and np.array_equal(a.ids, b[1])
        ls = kf.build_ls_coefficients(c)
        wx, wy, _ = r.ls_full()
        assert np.array_equal(ls.full_wx, wx) and np.array_equal(ls.full_wy, wy)
        assert np.array_equal(kf.color_points(c).color, r.colors())
    # a saved-and-loaded generated cloud equals the reference's load_cloud
    a = kf.generate_naca_ogrid("2412", 65, 9, 11.0)
    path = tmp_path / "c.txt"
    kf.save_cloud(a, path)
    r = Reference.load(path)
    x, y, kind, nx, ny = r.geometry()
    b = kf.load_cloud(path)
    assert np.array_equal(b.x, x) and np.array_equal(b.normal_y, ny)

"""Mesh import (bte_mesh_read: Gmsh ASCII 2.2 / 4.1, MEDIT) and recursive
coordinate bisection (bte_partition_rcb) -- SURVEY 8(f) f3; P:L544-547 (mesh
import), P:L589-592 (mesh partitioning).  Host-only library calls: run on CPU.

The writers below are written here from the two file formats' published
layouts, independently of the library's reader; coordinates go out as
repr() strings, so a correct reader returns the generator's arrays bit for bit."""
import os

import numpy as np
import pytest

import bte_inputs as bi
from paper_2305_19400_b200 import BteError, partition_rcb, plan_umesh, read_mesh

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _etype(m):
    return {3: 2, 4: 3 if m.dim == 2 else 4, 8: 5}[m.cells.shape[1]]


def _gmsh22(path, m, extra_boundary=True):
    etype = _etype(m)
    with open(path, "w") as f:
        f.write("$MeshFormat\n2.2 0 8\n$EndMeshFormat\n$Nodes\n%d\n" % m.nverts)
        for k, x in enumerate(m.verts):
            f.write("%d %s %s %s\n" % (k + 1, repr(float(x[0])), repr(float(x[1])), repr(float(x[2]))))
        f.write("$EndNodes\n$Elements\n")
        recs = []
        if extra_boundary:  # a point and a line: boundary tags the reader must skip
            recs.append("15 2 0 1 1")
            recs.append("1 2 3 1 1 2")
        for c in m.cells:
            recs.append("%d 2 0 3 %s" % (etype, " ".join(str(int(v) + 1) for v in c)))
        f.write("%d\n" % len(recs))
        for k, r in enumerate(recs):
            f.write("%d %s\n" % (k + 1, r))
        f.write("$EndElements\n")


def _gmsh41(path, m):
    etype = _etype(m)
    n = m.nverts
    half = n // 2
    with open(path, "w") as f:
        f.write("$MeshFormat\n4.1 0 8\n$EndMeshFormat\n")
        f.write("$Nodes\n2 %d 1 %d\n" % (n, n))
        for lo, hi in ((0, half), (half, n)):
            f.write("%d 1 0 %d\n" % (m.dim, hi - lo))
            for k in range(lo, hi):
                f.write("%d\n" % (k + 1))
            for k in range(lo, hi):
                x = m.verts[k]
                f.write("%s %s %s\n" % (repr(float(x[0])), repr(float(x[1])), repr(float(x[2]))))
        f.write("$EndNodes\n$Elements\n1 %d 1 %d\n%d 1 %d %d\n" % (m.ncells, m.ncells, m.dim, etype, m.ncells))
        for k, c in enumerate(m.cells):
            f.write("%d %s\n" % (k + 1, " ".join(str(int(v) + 1) for v in c)))
        f.write("$EndElements\n")


def _medit(path, m):
    kw = {3: "Triangles", 4: "Quadrilaterals" if m.dim == 2 else "Tetrahedra", 8: "Hexahedra"}[m.cells.shape[1]]
    with open(path, "w") as f:
        f.write("MeshVersionFormatted 2\n# written by the tests\nDimension %d\nVertices\n%d\n" % (m.dim, m.nverts))
        for x in m.verts:
            f.write(" ".join(repr(float(v)) for v in x[:m.dim]) + " 0\n")
        if m.dim == 3:  # boundary triangles the reader must treat as tags
            f.write("Triangles\n1\n1 2 3 5\n")
        f.write("%s\n%d\n" % (kw, m.ncells))
        for c in m.cells:
            f.write(" ".join(str(int(v) + 1) for v in c) + " 0\n")
        f.write("End\n")


@pytest.mark.parametrize("name", ["square_2tri_gmsh22.msh", "square_2tri_gmsh41.msh", "square_2tri.mesh"])
def test_golden_fixtures(name):
    m = read_mesh(os.path.join(GOLD, name))
    assert m.dim == 2 and m.cells.shape == (2, 3)
    np.testing.assert_array_equal(m.verts, [[0, 0, 0], [2e-6, 0, 0], [2e-6, 1e-6, 0], [0, 1e-6, 0]])
    np.testing.assert_array_equal(m.cells, [[0, 1, 2], [0, 2, 3]])


def _meshes():
    return {"tri": bi.umesh_tri(5, 4, 5e-6, 4e-6, jitter=0.2, seed=3, shuffle=True),
            "quad": bi.umesh_quad(4, 3, 4e-6, 3e-6, jitter=0.2, seed=4),
            "tet": bi.umesh_tet(3, 3, 2, 1e-6, jitter=0.1, seed=5, shuffle=True),
            "hex": bi.umesh_hex(3, 2, 2, 1e-6, jitter=0.1, seed=6, shuffle=True)}


@pytest.mark.parametrize("fmt", ["gmsh22", "gmsh41", "medit"])
@pytest.mark.parametrize("kind", ["tri", "quad", "tet", "hex"])
def test_roundtrip_bit_exact(tmp_path, fmt, kind):
    m = _meshes()[kind]
    path = str(tmp_path / ("m.mesh" if fmt == "medit" else "m.msh"))
    {"gmsh22": _gmsh22, "gmsh41": _gmsh41, "medit": _medit}[fmt](path, m)
    r = read_mesh(path, depth=m.depth)
    assert r.dim == m.dim
    np.testing.assert_array_equal(r.verts, m.verts)
    np.testing.assert_array_equal(r.cells, m.cells)


def test_read_errors(tmp_path):
    with pytest.raises(BteError, match="cannot open"):
        read_mesh(str(tmp_path / "missing.msh"))
    bad = tmp_path / "bin.msh"
    bad.write_text("$MeshFormat\n2.2 1 8\n$EndMeshFormat\n")
    with pytest.raises(BteError, match="binary"):
        read_mesh(str(bad))
    prism = tmp_path / "prism.msh"
    prism.write_text("$MeshFormat\n2.2 0 8\n$EndMeshFormat\n$Nodes\n6\n" +
                     "".join("%d %d %d %d\n" % (k + 1, k & 1, (k >> 1) & 1, k >> 2) for k in range(6)) +
                     "$EndNodes\n$Elements\n1\n1 6 0 1 2 3 4 5 6\n$EndElements\n")
    with pytest.raises(BteError, match="not supported"):
        read_mesh(str(prism))
    mixed = tmp_path / "mixed.mesh"
    mixed.write_text("MeshVersionFormatted 2\nDimension 2\nVertices\n4\n0 0 0\n1 0 0\n1 1 0\n0 1 0\n"
                     "Triangles\n1\n1 2 3 0\nQuadrilaterals\n1\n1 2 3 4 0\nEnd\n")
    with pytest.raises(BteError, match="mixed"):
        read_mesh(str(mixed))
    oob = tmp_path / "oob.mesh"
    oob.write_text("MeshVersionFormatted 2\nDimension 2\nVertices\n3\n0 0 0\n1 0 0\n1 1 0\nTriangles\n1\n1 2 9 0\nEnd\n")
    with pytest.raises(BteError, match="out of range"):
        read_mesh(str(oob))


def _centroids(m):
    return m.verts[m.cells].mean(axis=1)


@pytest.mark.parametrize("kind,P", [("tri", 3), ("tri", 8), ("tet", 4), ("tet", 7), ("hex", 5)])
def test_rcb_parts_are_ranges_compact_and_cut_halos(kind, P):
    """RCB on a randomly ordered mesh: a permutation; part r is exactly the
    range bte_create_umesh gives rank r; parts are compact (their centroid
    boxes overlap little); halos far smaller than for the shuffled order."""
    if kind == "tri":
        m = bi.umesh_tri(24, 20, 24e-6, 20e-6, jitter=0.2, seed=8, shuffle=True)
    elif kind == "hex":
        m = bi.umesh_hex(12, 10, 9, 1e-6, jitter=0.1, seed=10, shuffle=True)
    else:
        m = bi.umesh_tet(8, 7, 6, 1e-6, jitter=0.1, seed=9, shuffle=True)
    perm = partition_rcb(m, P)
    assert np.array_equal(np.sort(perm), np.arange(m.ncells))
    assert np.array_equal(perm, partition_rcb(m, P))  # deterministic
    mp = bi.UMesh(m.dim, m.verts, np.ascontiguousarray(m.cells[perm]), m.depth)
    cen = _centroids(mp)
    n = m.ncells
    vol = 0.0
    for r in range(P):
        lo, hi = r * n // P, (r + 1) * n // P
        c = cen[lo:hi]
        ext = c.max(0) - c.min(0)
        vol += np.prod(ext[:m.dim])
        assert np.all(np.diff(perm[lo:hi]) > 0)  # input order inside a part
    full = np.prod((cen.max(0) - cen.min(0))[:m.dim])
    assert vol < 1.35 * full, vol / full
    halo_rcb = sum(plan_umesh(mp, P, r)["n_halo"] for r in range(P))
    halo_shuf = sum(plan_umesh(m, P, r)["n_halo"] for r in range(P))
    assert halo_rcb < 0.25 * halo_shuf, (halo_rcb, halo_shuf)


def test_rcb_errors():
    m = bi.umesh_tri(3, 3, 3e-6, 3e-6)
    with pytest.raises(BteError):
        partition_rcb(m, 0)
    with pytest.raises(BteError):
        partition_rcb(m, m.ncells + 1)
    assert np.array_equal(partition_rcb(m, 1), np.arange(m.ncells))

"""Exact-rational (``fractions.Fraction``) twin of ONE explicit step -- TEST
INFRASTRUCTURE ONLY (pins the C oracle's sweep; pure-Python loops, tiny
meshes only).

Written from the face-sum definition rather than the oracle's per-axis
difference form, so that a dropped term, a wrong sign or a wrong neighbour in
either is caught:

  Eq. 5 + forward Euler, Eq. 3:
    I' = I + dt*( (I0 - I)*beta  -  v_b * (1/V) * sum_f A_f (s_d . n_f) I_up(f) )
  upwind: I_up = value in CELL1 (this cell) if s.n > 0, else the
    value in CELL2 (neighbour or ghost across f)  -- strict ">".
  ghosts (Eq. 6; reading #11 for diffuse walls).

Only LINEAR-mode channel tables are supported (I0 is then rational).
"""
from __future__ import annotations

from fractions import Fraction as Fr

import numpy as np


def _reflect_map(s, axis):
    nd = s.shape[0]
    r = []
    for d in range(nd):
        t = s[d].copy()
        t[axis] = -t[axis]
        hit = [e for e in range(nd) if np.array_equal(s[e], t)]
        if not hit:
            raise ValueError("reflection not closed")
        r.append(hit[0])
    return r


def exact_step_sweep(problem, I, I0c, betac):
    """One sweep step in exact rationals; returns an object array of Fractions [nc, nd, nb]."""
    m, dr, bd = problem.mesh, problem.dirs, problem.bands
    assert bd.mode == 0, "exact twin supports LINEAR channels only"
    nx, ny, nz = m.nx, m.ny, m.nz
    nd, nb = dr.nd, bd.nb
    dims = 3 if m.dim == 3 else 2
    D = [Fr(m.dx), Fr(m.dy), Fr(m.dz)]
    n = [nx, ny, nz]
    vol = D[0] * D[1] * D[2]
    s = [[Fr(float(x)) for x in row] for row in dr.s]
    w = [Fr(float(x)) for x in dr.w]
    v = [Fr(float(x)) for x in bd.v]
    dt = Fr(problem.dt)
    If = np.vectorize(Fr, otypes=[object])(np.asarray(I, dtype=np.float64))
    I0f = np.vectorize(Fr, otypes=[object])(np.asarray(I0c, dtype=np.float64))
    bf = np.vectorize(Fr, otypes=[object])(np.asarray(betac, dtype=np.float64))
    refl = {a: _reflect_map(dr.s, a) for a in range(dims)}

    def cidx(x, y, z):
        return x + nx * (y + ny * z)

    def I0_lin(b, T):
        return Fr(float(bd.I_ref[b])) + Fr(float(bd.slope[b])) * (Fr(float(T)) - Fr(float(bd.T_ref)))

    def ghost(region, ijk, d, b):
        a = region // 2
        bc = problem.bcs[region]
        c = cidx(*ijk)
        if bc.kind == 0:  # isothermal: I0_b(T_wall) at the face
            if bc.T_wall is None:
                T = bc.T_uniform
            else:
                f = [ijk[1] + ny * ijk[2], ijk[0] + nx * ijk[2], ijk[0] + nx * ijk[1]][a]
                T = bc.T_wall[f]
            return I0_lin(b, T)
        if bc.kind == 1:  # specular
            return If[c, refl[a][d], b]
        sg = 1 if region & 1 else -1  # diffuse: outgoing re-emitted isotropically
        num = sum((w[e] * abs(s[e][a]) * If[c, e, b] for e in range(nd) if sg * s[e][a] > 0), Fr(0))
        den = sum((w[e] * abs(s[e][a]) for e in range(nd) if sg * s[e][a] < 0), Fr(0))
        return num / den

    out = np.empty((nx * ny * nz, nd, nb), dtype=object)
    for z in range(nz):
        for y in range(ny):
            for x in range(nx):
                ijk = (x, y, z)
                c = cidx(x, y, z)
                for d in range(nd):
                    for b in range(nb):
                        face_sum = Fr(0)
                        for a in range(dims):
                            area = vol / D[a]
                            for side in (-1, +1):  # face on the -a / +a side of the cell
                                sn = s[d][a] * side  # s . n with n = side * e_a
                                if sn > 0:
                                    up = If[c, d, b]
                                else:
                                    nb_ijk = list(ijk)
                                    nb_ijk[a] += side
                                    if 0 <= nb_ijk[a] < n[a]:
                                        up = If[cidx(*nb_ijk), d, b]
                                    else:
                                        up = ghost(2 * a + (1 if side > 0 else 0), ijk, d, b)
                                face_sum += area * sn * up
                        out[c, d, b] = If[c, d, b] + dt * ((I0f[c, b] - If[c, d, b]) * bf[c, b]
                                                            - v[b] * face_sum / vol)
    return out


def ulp_error(approx, exact):
    """max |approx - exact| in units of ulp(exact) (exact: Fraction array)."""
    worst = 0.0
    for a, e in zip(np.asarray(approx).reshape(-1), exact.reshape(-1)):
        ef = float(e)
        u = np.spacing(abs(ef)) if ef != 0 else np.finfo(float).tiny
        err = abs(Fr(float(a)) - e)
        worst = max(worst, float(err / Fr(u)))
    return worst


def exact_usweep(problem, I, I0c, betac):
    """One sweep step on an UNSTRUCTURED simplex mesh in exact rationals
    (SURVEY 8(f) f3), written from Eq. 3 with rational geometry:
    for a face f of cell c, A_f n_f / V_c is computed without square roots --
      triangle: A_f n_f = depth * perp(edge), V = depth * |cross| / 2,
      tetrahedron: A_f n_f = cross(b - a, c - a) / 2, V = |det| / 6,
    oriented away from the opposite vertex;
      hexahedron (8 vertices, Gmsh order): face = bilinear patch through its
      4 corners q0..q3, A_f n_f = cross(q2 - q0, q3 - q1) / 2 (the integral of
      the normal over the patch), oriented away from the vertex mean;
      V = sum_f qbar_f . A_f n_f / 3 (divergence theorem, exact for such
      faces; qbar_f the mean of the face's corners).  Faces are matched by their vertex
    sets; a boundary face's wall is the box plane all its vertices lie on.
    Returns Fractions [nc, nd, nb].  LINEAR channel tables only."""
    m, dr, bd = problem.mesh, problem.dirs, problem.bands
    assert bd.mode == 0, "exact twin supports LINEAR channels only"
    nd, nb = dr.nd, bd.nb
    hexa = m.dim == 3 and int(m.cells.shape[1]) == 8
    HEXF = ((0, 1, 2, 3), (4, 5, 6, 7), (0, 1, 5, 4), (1, 2, 6, 5), (2, 3, 7, 6), (3, 0, 4, 7))
    K = 6 if hexa else int(m.cells.shape[1])
    P = [[Fr(float(x)) for x in row] for row in m.verts]
    cells = [[int(v) for v in row] for row in m.cells]
    nc = len(cells)
    lo = [min(p[a] for p in P) for a in range(3)]
    hi = [max(p[a] for p in P) for a in range(3)]
    s = [[Fr(float(x)) for x in row] for row in dr.s]
    w = [Fr(float(x)) for x in dr.w]
    v = [Fr(float(x)) for x in bd.v]
    dt = Fr(problem.dt)
    depth = Fr(float(m.depth))
    If = np.vectorize(Fr, otypes=[object])(np.asarray(I, dtype=np.float64))
    I0f = np.vectorize(Fr, otypes=[object])(np.asarray(I0c, dtype=np.float64))
    bf = np.vectorize(Fr, otypes=[object])(np.asarray(betac, dtype=np.float64))
    refl = {a: _reflect_map(dr.s, a) for a in range(m.dim)}
    def face_verts(cv, k):  # 2-D: edge (v_{k+1}, v_{k+2}); 3-D: the face opposite v_k; hexahedron: HEXF[k]
        if hexa:
            return [cv[i] for i in HEXF[k]]
        if m.dim == 2:
            return [cv[(k + 1) % K], cv[(k + 2) % K]]
        return cv[:k] + cv[k + 1:]

    owner = {}
    for c, cv in enumerate(cells):
        for k in range(K):
            owner.setdefault(frozenset(face_verts(cv, k)), []).append((c, k))
    # wall faces in (cell, local face) order per region
    wall_index = {}
    count = [0] * 6

    def sub(p, q):
        return [p[i] - q[i] for i in range(3)]

    def dot(p, q):
        return p[0] * q[0] + p[1] * q[1] + p[2] * q[2]

    geo = []  # per cell: volume, [(An vector, neighbour or None, region)]
    for c, cv in enumerate(cells):
        X = [P[i] for i in cv]
        if hexa:
            cm = [sum((X[k][a] for k in range(8)), Fr(0)) / 8 for a in range(3)]
            V = Fr(0)
            hexS = []
            for k in range(6):
                q = [X[i] for i in HEXF[k]]
                d1, d2 = sub(q[2], q[0]), sub(q[3], q[1])
                S = [(d1[1] * d2[2] - d1[2] * d2[1]) / 2, (d1[2] * d2[0] - d1[0] * d2[2]) / 2,
                     (d1[0] * d2[1] - d1[1] * d2[0]) / 2]
                qb = [(q[0][a] + q[1][a] + q[2][a] + q[3][a]) / 4 for a in range(3)]
                if dot(S, sub(qb, cm)) < 0:
                    S = [-x for x in S]
                V += dot(qb, S) / 3
                hexS.append(S)
        elif m.dim == 2:  # shoelace (for a triangle: |cross| / 2)
            sh = sum((X[k][0] * X[(k + 1) % K][1] - X[(k + 1) % K][0] * X[k][1] for k in range(K)), Fr(0))
            V = abs(sh) / 2 * depth
            cen = [sum((X[k][a] for k in range(K)), Fr(0)) / K for a in range(3)]
        else:
            u, vv, ww = sub(X[1], X[0]), sub(X[2], X[0]), sub(X[3], X[0])
            det = (u[0] * (vv[1] * ww[2] - vv[2] * ww[1]) - u[1] * (vv[0] * ww[2] - vv[2] * ww[0])
                   + u[2] * (vv[0] * ww[1] - vv[1] * ww[0]))
            V = abs(det) / 6
        faces = []
        for k in range(K):
            if hexa:
                others = [P[v] for v in face_verts(cv, k)]
                An = hexS[k]
            elif m.dim == 2:
                others = [P[v] for v in face_verts(cv, k)]
                e = sub(others[1], others[0])
                An = [e[1] * depth, -e[0] * depth, Fr(0)]
                if dot(An, sub(cen, others[0])) > 0:  # outward: away from the vertex mean
                    An = [-x for x in An]
            else:
                others = [X[i] for i in range(K) if i != k]
                e1, e2 = sub(others[1], others[0]), sub(others[2], others[0])
                An = [(e1[1] * e2[2] - e1[2] * e2[1]) / 2, (e1[2] * e2[0] - e1[0] * e2[2]) / 2,
                      (e1[0] * e2[1] - e1[1] * e2[0]) / 2]
                if dot(An, sub(X[k], others[0])) > 0:
                    An = [-x for x in An]
            key = frozenset(face_verts(cv, k))
            nbr = [o for o in owner[key] if o[0] != c]
            region = None
            if not nbr:
                for r in range(2 * m.dim):
                    a = r // 2
                    wall = hi[a] if r & 1 else lo[a]
                    if all(p[a] == wall for p in others):
                        region = r
                        break
                assert region is not None, "boundary face off the box walls"
                wall_index[(c, k)] = count[region]
                count[region] += 1
            faces.append((An, nbr[0][0] if nbr else None, region))
        geo.append((V, faces))

    def I0_lin(b, T):
        return Fr(float(bd.I_ref[b])) + Fr(float(bd.slope[b])) * (Fr(float(T)) - Fr(float(bd.T_ref)))

    def ghost(region, c, k, d, b):
        a = region // 2
        bc = problem.bcs[region]
        if bc.kind == 0:
            T = bc.T_uniform if bc.T_wall is None else bc.T_wall[wall_index[(c, k)]]
            return I0_lin(b, T)
        spec = If[c, refl[a][d], b] if bc.kind in (1, 3) else None
        if bc.kind == 1:
            return spec
        sg = 1 if region & 1 else -1
        num = sum((w[e] * abs(s[e][a]) * If[c, e, b] for e in range(nd) if sg * s[e][a] > 0), Fr(0))
        den = sum((w[e] * abs(s[e][a]) for e in range(nd) if sg * s[e][a] < 0), Fr(0))
        diff = num / den
        if bc.kind == 2:
            return diff
        p = Fr(float(bc.specularity))
        return p * spec + (1 - p) * diff

    out = np.empty((nc, nd, nb), dtype=object)
    for c in range(nc):
        V, faces = geo[c]
        for d in range(nd):
            for b in range(nb):
                face_sum = Fr(0)
                for k, (An, nbr, region) in enumerate(faces):
                    sAn = dot(s[d], An)
                    if sAn > 0:
                        up = If[c, d, b]
                    elif nbr is not None:
                        up = If[nbr, d, b]
                    else:
                        up = ghost(region, c, k, d, b)
                    face_sum += sAn * up
                out[c, d, b] = If[c, d, b] + dt * ((I0f[c, b] - If[c, d, b]) * bf[c, b] - v[b] * face_sum / V)
    return out

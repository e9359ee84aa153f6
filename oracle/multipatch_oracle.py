"""CPU restatement of the multipatch extension (BASELINE cfg4) -- TEST
INFRASTRUCTURE ONLY (imported by tests/, never by the product).

PARITY UNPINNED: the reference has no multipatch code path (SPEC.md:150,208,
SURVEY.md 8(c)); this oracle restates, independently of the device code,
the extension DESIGN.md describes: per-patch full stiffness by element
quadrature (basis tables from the C oracle's restatement of
assembly.py:209-234, geometry from its NurbsPatch.eval_grid restatement),
C0 gluing of conforming interfaces, Dirichlet values by L2 projection onto
the boundary trace space, dense solves of the lifted interior system.
"""
from __future__ import annotations

import numpy as np

from oracle import oracle as O
from paper_1707_09598_b200.pipeline import gauss_rule


def _dir_tables(kv, regularity, q):
    gn, gw = gauss_rule(q)
    return O.direction_tables(kv.degree, regularity, kv.breakpoints, q, gn, gw)


def _geometry(orc, pts_per_dir):
    x, J, det, code = orc.geometry_grid(pts_per_dir)
    if code != 0:
        raise ValueError("degenerate geometry")
    return x, J, det


def patch_system(orc, kvs, regularity, q, forcing):
    """Full stiffness (dense, C-order dofs) and load vector of one 2-D patch."""
    tabs = [_dir_tables(kv, regularity, q) for kv in kvs]
    n = [kv.knots.size - kv.degree - 1 for kv in kvs]
    P = kvs[0].degree + 1
    (vx, dx, ox, px, wx), (vy, dy, oy, py, wy) = tabs
    x, J, det = _geometry(orc, (px, py))
    nqx, nqy = px.size, py.size
    Jinv = np.linalg.inv(J)
    w = np.outer(wx, wy).ravel()
    G = np.einsum("nmi,nki->nmk", Jinv, Jinv) * (det * w)[:, None, None]
    L = forcing(x) * det * w
    G = G.reshape(nqx, nqy, 2, 2)
    L = L.reshape(nqx, nqy)
    N = n[0] * n[1]
    A = np.zeros((N, N))
    b = np.zeros(N)
    nelx, nely, q_ = vx.shape[0], vy.shape[0], vx.shape[1]
    for ex in range(nelx):
        for ey in range(nely):
            sx, sy = slice(ex * q_, ex * q_ + q_), slice(ey * q_, ey * q_ + q_)
            Ge, Le = G[sx, sy], L[sx, sy]                     # [qx, qy, 2, 2], [qx, qy]
            # local basis products: grad N_(a,b) at (gx, gy)
            Bx, Dx, By, Dy = vx[ex], dx[ex], vy[ey], dy[ey]   # [q, P]
            grad = np.stack([np.einsum("ia,jb->ijab", Dx, By), np.einsum("ia,jb->ijab", Bx, Dy)], axis=-1)
            val = np.einsum("ia,jb->ijab", Bx, By)
            Ke = np.einsum("ijabm,ijmn,ijcdn->abcd", grad, Ge, grad).reshape(P * P, P * P)
            be = np.einsum("ijab,ij->ab", val, Le).reshape(P * P)
            gi = ((ox[ex] + np.arange(P))[:, None] * n[1] + (oy[ey] + np.arange(P))[None, :]).ravel()
            A[np.ix_(gi, gi)] += Ke
            b[gi] += be
    return A, b, n


def edge_system(orc, kv_edge, regularity, q, edge_axis, side, g):
    """1-D mass and data moments on one patch edge (L2 on the physical edge)."""
    vals, ders, offs, pts, wts = _dir_tables(kv_edge, regularity, q)
    grid = [None, None]
    grid[edge_axis] = pts
    grid[1 - edge_axis] = np.array([float(side)])
    x, J, det = _geometry(orc, tuple(grid))
    tang = J[:, :, edge_axis]
    jac = np.sqrt((tang * tang).sum(axis=1))
    n = kv_edge.knots.size - kv_edge.degree - 1
    P = kv_edge.degree + 1
    M, r = np.zeros((n, n)), np.zeros(n)
    gv = g(x)
    nel, q_ = vals.shape[0], vals.shape[1]
    for e in range(nel):
        sl = slice(e * q_, e * q_ + q_)
        wj = wts[sl] * jac[sl]
        idx = offs[e] + np.arange(P)
        M[np.ix_(idx, idx)] += np.einsum("ia,ib,i->ab", vals[e], vals[e], wj)
        r[idx] += np.einsum("ia,i->a", vals[e], gv[sl] * wj)
    return M, r


def solve_component(specs, problem, comp, q):
    """Per-patch full coefficient vectors of one component (list, C order)."""
    npatch = len(specs)
    orcs = [O.Oracle(s) for s in specs]
    kvs = []
    for pi, s in enumerate(specs):
        beta = s.terms[comp][0]
        kvs.append([problem.knot_rules[pi](k, int(lv)) for k, lv in enumerate(beta)])
    systems = [patch_system(orcs[pi], kvs[pi], problem.regularity, q, problem.forcing) for pi in range(npatch)]
    dims = [sys[2] for sys in systems]
    base = np.concatenate([[0], np.cumsum([a * b for a, b in dims])])
    # independent global numbering: follow the interfaces explicitly
    label = np.arange(base[-1])

    def side(pi, axis, s):
        nx, ny = dims[pi]
        if axis == 0:
            i = nx - 1 if s else 0
            return base[pi] + i * ny + np.arange(ny)
        j = ny - 1 if s else 0
        return base[pi] + np.arange(nx) * ny + j

    changed = True
    pairs = [(side(f.a, f.a_axis, f.a_side), side(f.b, f.b_axis, f.b_side)) for f in problem.interfaces]
    while changed:
        changed = False
        for la, lb in pairs:
            m = np.minimum(label[la], label[lb])
            if np.any(m != label[la]) or np.any(m != label[lb]):
                label[la] = m
                label[lb] = m
                changed = True
    iface = {(f.a, f.a_axis, f.a_side) for f in problem.interfaces} | \
            {(f.b, f.b_axis, f.b_side) for f in problem.interfaces}
    dsides = [(pi, ax, s) for pi in range(npatch) for ax in (0, 1) for s in (0, 1) if (pi, ax, s) not in iface]
    is_dir = np.zeros(base[-1], dtype=bool)
    for pi, ax, s in dsides:
        is_dir[side(pi, ax, s)] = True
    roots = np.unique(label)
    root_dir = {int(r): False for r in roots}
    for i in range(base[-1]):
        if is_dir[i]:
            root_dir[int(label[i])] = True
    inter = [r for r in roots if not root_dir[int(r)]]
    bnd = [r for r in roots if root_dir[int(r)]]
    pos = {int(r): k for k, r in enumerate(inter)}
    bpos = {int(r): k for k, r in enumerate(bnd)}
    nI, nB = len(inter), len(bnd)
    AII, AIB, bI = np.zeros((nI, nI)), np.zeros((nI, nB)), np.zeros(nI)
    for pi in range(npatch):
        A, b, _ = systems[pi]
        lab = label[base[pi]:base[pi + 1]]
        for r_ in range(A.shape[0]):
            gr = int(lab[r_])
            if gr not in pos:
                continue
            bI[pos[gr]] += b[r_]
            for c_ in np.nonzero(A[r_])[0]:
                gc = int(lab[c_])
                if gc in pos:
                    AII[pos[gr], pos[gc]] += A[r_, c_]
                else:
                    AIB[pos[gr], bpos[gc]] += A[r_, c_]
    MBB, rB = np.zeros((nB, nB)), np.zeros(nB)
    for pi, ax, s in dsides:
        eaxis = 1 - ax
        M, r = edge_system(orcs[pi], kvs[pi][eaxis], problem.regularity, q, eaxis, s, problem.dirichlet)
        loc = [bpos[int(label[i])] for i in side(pi, ax, s)]
        MBB[np.ix_(loc, loc)] += M
        rB[loc] += r
    uB = np.linalg.solve(MBB, rB)
    uI = np.linalg.solve(AII, bI - AIB @ uB)
    out = []
    for pi in range(npatch):
        lab = label[base[pi]:base[pi + 1]]
        out.append(np.array([uI[pos[int(l_)]] if int(l_) in pos else uB[bpos[int(l_)]] for l_ in lab]))
    return out


def run_plan(specs, problem, q):
    """Per-patch concatenated full coefficients (plan order) for every patch."""
    ncomp = len(specs[0].terms)
    per = [solve_component(specs, problem, c, q) for c in range(ncomp)]
    return [np.concatenate([per[c][pi] for c in range(ncomp)]) for pi in range(len(specs))]

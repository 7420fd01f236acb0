"""Seeded adversarial families for the intersects culls.

Each family is built where the REFERENCE's own arithmetic is noisy, so that
it reports hits the exact geometry does not have (or misses ones it has):

* sliver_literal   : B = one sliver (|N| = w, K = |e0||e1|/|N| up to 1e13);
                     A = triangles with an edge whose endpoints sit 1e-12..1e-2
                     off the sliver's plane over the sliver (the reference's
                     t is noisy by ~3.6e-15 K D, advisor's case);
* sliver_records   : the same with the roles swapped (A = slivers near one
                     lifted edge of B);
* grazing_parallel : A's edge nearly parallel to B's plane (1e-12..1e-8 rad),
                     crossing it 1e-9..1e-2 outside B while B stays on one side
                     of A's plane (the reference's u, v are noisy ~1.8e-15/alpha);
* sliver_segments  : segments vs a mesh of slivers (segment queries).

Every family is placed by a random rigid motion, scale and offset.
old_cull_separates() models the round-1 cull (one-way plane test with
tau = 1e-10 D + 1e-13 max|coord|, either direction) so the CPU test can show
the families contain reference hits that cull dropped.
"""
import numpy as np


def _rot(rng):
    q, r = np.linalg.qr(rng.normal(size=(3, 3)))
    return q * np.sign(np.diag(r))[None, :]


def place(rng, *meshes, big=False):
    """One shared rigid motion + scale + offset for all the given (n, 9|6) arrays."""
    R = _rot(rng)
    s = 10.0 ** rng.integers(-2, 3)
    t = rng.uniform(-1, 1, 3) * (1e5 if big else 3.0)
    out = []
    for m in meshes:
        w = m.shape[1]
        out.append(np.ascontiguousarray(((m.reshape(-1, 3) @ R.T) * s + t).reshape(-1, w)))
    return out


def sliver(w, length=1.0):
    return np.array([[0.0, 0.0, 0.0, length, 0.0, 0.0, 0.5 * length, w, 0.0]])


def lifted_edges(rng, n, x_lo=-0.1, x_hi=1.1, y_scale=1e-6):
    """Triangles (P, Q, R) with P, Q just off z = 0 (heights 1e-12..1e-2, same or
    opposite sides), over the strip |y| <= y_scale, R far above."""
    P = np.stack([rng.uniform(x_lo, x_hi, n), rng.normal(scale=y_scale, size=n),
                  10.0 ** rng.uniform(-12, -2, n) * rng.choice([-1, 1], n)], 1)
    Q = np.stack([rng.uniform(x_lo, x_hi, n), rng.normal(scale=y_scale, size=n),
                  10.0 ** rng.uniform(-12, -2, n) * rng.choice([-1, 1], n)], 1)
    R = np.stack([rng.uniform(-1, 2, n), rng.uniform(-1, 1, n), rng.uniform(0.3, 1.0, n) * rng.choice([-1, 1], n)], 1)
    return np.concatenate([P, Q, R], 1)


def sliver_literal(rng, n, w):
    lit = sliver(w)
    recs = lifted_edges(rng, n, y_scale=max(w, 1e-12) * 2)
    lit, recs = place(rng, lit, recs, big=rng.random() < 0.3)
    return recs, lit


def sliver_records(rng, n):
    """Slivers (w = 1e-13..1e-6, random length and position) under one lifted edge."""
    lit = np.array([[0.2, 0.0, 3e-9, 0.8, 0.0, -2e-9, 0.5, 0.4, 0.9]])
    w = 10.0 ** rng.uniform(-13, -6, n)
    x0 = rng.uniform(-0.2, 0.6, n)
    L = rng.uniform(0.2, 1.0, n)
    y0 = rng.normal(scale=1e-7, size=n)
    z0 = 10.0 ** rng.uniform(-12, -3, n) * rng.choice([-1, 1], n)
    recs = np.stack([x0, y0, z0, x0 + L, y0, z0, x0 + 0.5 * L, y0 + w, z0], 1)
    tilt = 10.0 ** rng.uniform(-12, -4, n) * rng.choice([-1, 1], n)
    recs[:, 5] += tilt  # V1 slightly off the z = z0 plane
    lit, recs = place(rng, lit, recs, big=rng.random() < 0.3)
    return recs, lit


def grazing_parallel(rng, n):
    """B = a unit right triangle in z = 0. A = (P, Q, R): PQ crosses z = 0 at X,
    delta outside B's hypotenuse, at angle alpha to the plane, running along
    the hypotenuse; R straight above X so A's plane is near vertical and B lies
    on one side of it by ~delta."""
    lit = np.array([[0.0, 0.0, 0.0, 1.0, 0.0, 0.0, 0.0, 1.0, 0.0]])
    alpha = 10.0 ** rng.uniform(-12, -8, n)
    delta = 10.0 ** rng.uniform(-9, -2, n)
    s = rng.uniform(0.1, 0.9, n)                   # where along the hypotenuse
    tdir = np.array([-1.0, 1.0, 0.0]) / np.sqrt(2)  # hypotenuse direction
    out = np.array([1.0, 1.0, 0.0]) / np.sqrt(2)    # outward normal of the hypotenuse
    X = np.array([1.0, 0.0, 0.0]) + s[:, None] * np.sqrt(2) * tdir + delta[:, None] * out
    a0, a1 = rng.uniform(0.05, 0.5, n), rng.uniform(0.05, 0.5, n)
    d = tdir[None, :] + alpha[:, None] * np.array([0.0, 0.0, 1.0])
    P = X - a0[:, None] * d
    Q = X + a1[:, None] * d
    R = X + np.array([0.0, 0.0, 1.0]) + rng.normal(scale=1e-3, size=(n, 3)) * [1, 1, 0] + 0.3 * out
    recs = np.concatenate([P, Q, R], 1)
    lit, recs = place(rng, lit, recs, big=rng.random() < 0.3)
    return recs, lit


def sliver_mesh_and_segments(rng, n_faces, n_segs):
    """A soup of slivers (w = 1e-13..1e-7) along x, and segments whose
    endpoints sit 1e-12..1e-2 off the sliver planes over them."""
    x0 = rng.uniform(0, 10, n_faces)
    w = 10.0 ** rng.uniform(-13, -7, n_faces)
    y0 = rng.uniform(0, 10, n_faces)
    mesh = np.stack([x0, y0, np.zeros(n_faces), x0 + 1, y0, np.zeros(n_faces), x0 + 0.5, y0 + w,
                     np.zeros(n_faces)], 1)
    k = rng.integers(0, n_faces, n_segs)
    px = x0[k] + rng.uniform(-0.1, 1.1, n_segs)
    qx = x0[k] + rng.uniform(-0.1, 1.1, n_segs)
    yy = y0[k] + rng.normal(scale=1e-9, size=n_segs)
    h0 = 10.0 ** rng.uniform(-12, -2, n_segs) * rng.choice([-1, 1], n_segs)
    h1 = 10.0 ** rng.uniform(-12, -2, n_segs) * rng.choice([-1, 1], n_segs)
    segs = np.stack([px, yy, h0, qx, yy + rng.normal(scale=1e-9, size=n_segs), h1], 1)
    mesh, segs = place(rng, mesh, segs, big=rng.random() < 0.3)
    return mesh, segs


# ---- the round-1 cull, modelled in numpy (for the CPU demonstration) --------
def _plane(t):
    v0, v1, v2 = t[:, 0:3], t[:, 3:6], t[:, 6:9]
    N = np.cross(v1 - v0, v2 - v0)
    n = N / np.linalg.norm(N, axis=1, keepdims=True)
    return n, (n * v0).sum(1)


def old_cull_separates(a, b):
    """Round-1 hit_kernel: pair culled iff all three vertices of one triangle
    lie beyond tau = 1e-10 D + 1e-13 max|coord| on one side of the other's
    plane (either direction), D = diag of the pair's box."""
    allv = np.concatenate([a.reshape(-1, 3, 3), b.reshape(-1, 3, 3)], 1)
    D = np.linalg.norm(allv.max(1) - allv.min(1), axis=1)
    tau = 1e-10 * D + 1e-13 * np.abs(allv).max((1, 2))

    def sep(tri_plane, tri_pts):
        n, c = _plane(tri_plane)
        h = np.stack([(n * tri_pts[:, 3 * k:3 * k + 3]).sum(1) - c for k in range(3)], 1)
        return (h > tau[:, None]).all(1) | (h < -tau[:, None]).all(1)

    with np.errstate(invalid="ignore", divide="ignore"):
        return sep(b, a) | sep(a, b)


def kappa(t):
    """F_K of tdb_internal.h: 8e-15 |e0||e1| / |N| (+inf when N = 0)."""
    v0, v1, v2 = t[:, 0:3], t[:, 3:6], t[:, 6:9]
    e0, e1 = v1 - v0, v2 - v0
    N = np.linalg.norm(np.cross(e0, e1), axis=1)
    with np.errstate(divide="ignore"):
        return np.where(N > 0, 8e-15 * np.linalg.norm(e0, axis=1) * np.linalg.norm(e1, axis=1) / N, np.inf)


def new_cull_separates(a, b):
    """The round-2 culls (tdb_internal.h) at pair level (D = the pair's own box
    diagonal, the tightest D the device may use): one-way with
    (kCullOne + kappa) D, two-way with (kCullTwo + kappa) D, apart with kApart D."""
    allv = np.concatenate([a.reshape(-1, 3, 3), b.reshape(-1, 3, 3)], 1)
    D = np.linalg.norm(allv.max(1) - allv.min(1), axis=1)
    ab = 1e-13 * np.abs(allv).max((1, 2))
    ka, kb = kappa(a), kappa(b)
    A, B = a.reshape(-1, 3, 3), b.reshape(-1, 3, 3)
    gap = 5e-2 * D + ab
    apart = ((A.min(1) > B.max(1) + gap[:, None]) | (B.min(1) > A.max(1) + gap[:, None])).any(1)

    def heights(tri_plane, tri_pts):
        n, c = _plane(tri_plane)
        return np.stack([(n * tri_pts[:, 3 * k:3 * k + 3]).sum(1) - c for k in range(3)], 1)

    def sep(h, tau):
        return (h > tau[:, None]).all(1) | (h < -tau[:, None]).all(1)

    with np.errstate(invalid="ignore", divide="ignore", over="ignore"):
        hb = heights(a, b)  # B's vertices vs A's plane
        ha = heights(b, a)  # A's vertices vs B's plane
        one = sep(hb, (2.5e-2 + ka) * D + ab) | sep(ha, (2.5e-2 + kb) * D + ab)
        two = sep(hb, (1.01e-12 + ka) * D + ab) & sep(ha, (1.01e-12 + kb) * D + ab)
    return apart | one | two

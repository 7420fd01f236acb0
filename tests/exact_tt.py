"""Exact (rational) triangle-triangle distance, for the few pairs where the
reference's own FP64 composition is not the true distance (slivers, edges
parallel to the other plane below its 1e-12 threshold). Test-only checker:
every input double is an exact rational, every step is exact, so the result
is the true squared distance of the two closed triangles.
"""
from fractions import Fraction as Fr


def _v(p):
    return [Fr(float(x)) for x in p]


def _sub(a, b):
    return [a[0] - b[0], a[1] - b[1], a[2] - b[2]]


def _dot(a, b):
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]


def _cross(a, b):
    return [a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]]


def _clamp(x):
    return Fr(0) if x < 0 else Fr(1) if x > 1 else x


def point_segment2(p, a, b):
    d = _sub(b, a)
    L = _dot(d, d)
    t = Fr(0) if L == 0 else _clamp(_dot(_sub(p, a), d) / L)
    q = [a[i] + t * d[i] for i in range(3)]
    w = _sub(p, q)
    return _dot(w, w)


def segment_segment2(p0, p1, q0, q1):
    d1, d2, r = _sub(p1, p0), _sub(q1, q0), _sub(p0, q0)
    a, e, b = _dot(d1, d1), _dot(d2, d2), _dot(d1, d2)
    c, f = _dot(d1, r), _dot(d2, r)
    den = a * e - b * b
    best = min(point_segment2(p0, q0, q1), point_segment2(p1, q0, q1), point_segment2(q0, p0, p1),
               point_segment2(q1, p0, p1))
    if den != 0:
        s, t = (b * f - c * e) / den, (a * f - b * c) / den
        if 0 <= s <= 1 and 0 <= t <= 1:
            w = [p0[i] + s * d1[i] - q0[i] - t * d2[i] for i in range(3)]
            best = min(best, _dot(w, w))
    return best


def point_triangle2(p, t):
    v0, v1, v2 = t
    e0, e1 = _sub(v1, v0), _sub(v2, v0)
    N = _cross(e0, e1)
    NN = _dot(N, N)
    best = min(point_segment2(p, v0, v1), point_segment2(p, v1, v2), point_segment2(p, v2, v0))
    if NN != 0:
        w = _sub(p, v0)
        # barycentrics of the projection
        u = _dot(_cross(w, e1), N) / NN
        v = _dot(_cross(e0, w), N) / NN
        if u >= 0 and v >= 0 and u + v <= 1:
            h = _dot(w, N)
            best = min(best, h * h / NN)
    return best


def _orient(a, b, c, d):
    return _dot(_sub(b, a), _cross(_sub(c, a), _sub(d, a)))


def segment_crosses_triangle(p, q, t):
    v0, v1, v2 = t
    sp, sq = _orient(v0, v1, v2, p), _orient(v0, v1, v2, q)
    if sp == 0 and sq == 0:
        return False  # coplanar: distance via the boundary terms
    if (sp > 0 and sq > 0) or (sp < 0 and sq < 0):
        return False
    s0, s1, s2 = _orient(p, q, v0, v1), _orient(p, q, v1, v2), _orient(p, q, v2, v0)
    return (s0 >= 0 and s1 >= 0 and s2 >= 0) or (s0 <= 0 and s1 <= 0 and s2 <= 0)


def tri_tri_distance2(a9, b9):
    """True squared distance between two closed triangles (9 doubles each)."""
    A = [_v(a9[0:3]), _v(a9[3:6]), _v(a9[6:9])]
    B = [_v(b9[0:3]), _v(b9[3:6]), _v(b9[6:9])]
    for s, t in ((A, B), (B, A)):
        for k in range(3):
            if segment_crosses_triangle(s[k], s[(k + 1) % 3], t):
                return Fr(0)
    best = min(point_triangle2(p, B) for p in A)
    best = min(best, min(point_triangle2(p, A) for p in B))
    for i in range(3):
        for j in range(3):
            best = min(best, segment_segment2(A[i], A[(i + 1) % 3], B[j], B[(j + 1) % 3]))
    return best

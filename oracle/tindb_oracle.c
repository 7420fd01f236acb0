/* TEST INFRASTRUCTURE ONLY — see tindb_oracle.h.
 *
 * Restates the reference FP64 primitives in C, operation for operation, so
 * that results are bit-identical to the reference built without FMA
 * contraction (proj/CMakeLists.txt Release flags; x86-64 SSE2 scalar code).
 * Build with -ffp-contract=off (oracle/Makefile). Every expression keeps the
 * reference's left-to-right evaluation order; the citations give the
 * reference line each function follows.
 */
#include "tindb_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    double x, y, z;
} v3;

/* geometry.hpp:27-44 */
static inline v3 mk(double x, double y, double z) {
    v3 r = {x, y, z};
    return r;
}
static inline v3 ld3(const double* p) { return mk(p[0], p[1], p[2]); }
static inline v3 sub(v3 a, v3 b) { return mk(a.x - b.x, a.y - b.y, a.z - b.z); }
static inline v3 add(v3 a, v3 b) { return mk(a.x + b.x, a.y + b.y, a.z + b.z); }
static inline v3 scl(v3 a, double s) { return mk(a.x * s, a.y * s, a.z * s); }
static inline double dot3(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static inline v3 crs(v3 a, v3 b) {
    return mk(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
static inline double len(v3 a) { return sqrt(dot3(a, a)); }
static inline int same(v3 a, v3 b) { return a.x == b.x && a.y == b.y && a.z == b.z; }

static const double TINY = 1e-300;         /* kernels.cpp:50 kTiny */
static const double DEGEN_AREA2 = 1e-30;   /* geometry.hpp:58 */
static const double PIERCE_EPS = 1e-12;    /* kernels.hpp:53 */
static const double BARY_SLACK = 1e-12;    /* kernels.hpp:54 */

static inline double clamp_unit(double v) { return v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v); }

typedef struct {
    v3 v0, v1, v2;
} tri_t;

static inline tri_t ld_tri(const double* t) {
    tri_t r = {ld3(t), ld3(t + 3), ld3(t + 6)};
    return r;
}

/* geometry.hpp:75: norm2((v1-v0) x (v2-v0)) <= 1e-30 */
static inline int tri_degenerate(const tri_t* t) {
    v3 n = crs(sub(t->v1, t->v0), sub(t->v2, t->v0));
    return dot3(n, n) <= DEGEN_AREA2;
}

typedef struct {
    double d;
    v3 a, b;
} res_t;

/* kernels.cpp:54-60 make_pair_result: distance = |on_a - on_b| */
static inline res_t witness(v3 on_a, v3 on_b) {
    res_t r;
    r.a = on_a;
    r.b = on_b;
    r.d = len(sub(on_a, on_b));
    return r;
}

/* kernels.cpp:72-116 */
static res_t seg_seg(v3 a0, v3 a1, v3 b0, v3 b1) {
    const v3 d1 = sub(a1, a0), d2 = sub(b1, b0), r = sub(a0, b0);
    const double aa = dot3(d1, d1), ee = dot3(d2, d2), f = dot3(d2, r);
    double s = 0.0, t = 0.0;
    if (aa <= TINY && ee <= TINY) {
        /* two points */
    } else if (aa <= TINY) {
        t = clamp_unit(f / ee);
    } else {
        const double c = dot3(d1, r);
        if (ee <= TINY) {
            s = clamp_unit(-c / aa);
        } else {
            const double bb = dot3(d1, d2);
            const double den = aa * ee - bb * bb;
            if (den > TINY) s = clamp_unit((bb * f - c * ee) / den);
            t = (bb * s + f) / ee;
            if (t < 0.0) {
                t = 0.0;
                s = clamp_unit(-c / aa);
            } else if (t > 1.0) {
                t = 1.0;
                s = clamp_unit((bb - c) / aa);
            }
        }
    }
    return witness(add(a0, scl(d1, s)), add(b0, scl(d2, t)));
}

/* kernels.cpp:64-68 + :120-124 */
static res_t pt_seg(v3 p, v3 s0, v3 s1) {
    const v3 d = sub(s1, s0);
    const double dd = dot3(d, d);
    double t = 0.0;
    if (!(dd <= TINY)) t = clamp_unit(dot3(sub(p, s0), d) / dd);
    return witness(p, add(s0, scl(d, t)));
}

/* kernels.cpp:138-227 (degenerate fallback :127-134) */
static res_t pt_tri(v3 p, const tri_t* tr) {
    const v3 e0 = sub(tr->v1, tr->v0), e1 = sub(tr->v2, tr->v0), df = sub(tr->v0, p);
    const double a00 = dot3(e0, e0), a01 = dot3(e0, e1), a11 = dot3(e1, e1);
    const double b0 = dot3(df, e0), b1 = dot3(df, e1);
    const double det = a00 * a11 - a01 * a01;

    if (tri_degenerate(tr) || det <= TINY) {
        res_t best = pt_seg(p, tr->v0, tr->v1);
        res_t c = pt_seg(p, tr->v0, tr->v2);
        if (c.d < best.d) best = c;
        c = pt_seg(p, tr->v1, tr->v2);
        if (c.d < best.d) best = c;
        best.a = p;
        return best;
    }

    double s = a01 * b1 - a11 * b0;
    double t = a01 * b0 - a00 * b1;
    if (s + t <= det) {
        if (s < 0.0) {
            if (t < 0.0 && b0 < 0.0) { /* region 4, toward edge v0v1 */
                t = 0.0;
                s = -b0 >= a00 ? 1.0 : -b0 / a00;
            } else { /* region 4 (b0 >= 0) and region 3 share the v0v2 edge walk */
                s = 0.0;
                t = b1 >= 0.0 ? 0.0 : (-b1 >= a11 ? 1.0 : -b1 / a11);
            }
        } else if (t < 0.0) { /* region 5 */
            t = 0.0;
            s = b0 >= 0.0 ? 0.0 : (-b0 >= a00 ? 1.0 : -b0 / a00);
        } else { /* region 0 */
            s /= det;
            t /= det;
        }
    } else if (s < 0.0) { /* region 2 */
        const double q0 = a01 + b0, q1 = a11 + b1;
        if (q1 > q0) {
            const double num = q1 - q0, den = a00 - 2.0 * a01 + a11;
            s = num >= den ? 1.0 : num / den;
            t = 1.0 - s;
        } else {
            s = 0.0;
            t = q1 <= 0.0 ? 1.0 : (b1 >= 0.0 ? 0.0 : -b1 / a11);
        }
    } else if (t < 0.0) { /* region 6 */
        const double q0 = a01 + b1, q1 = a00 + b0;
        if (q1 > q0) {
            const double num = q1 - q0, den = a00 - 2.0 * a01 + a11;
            t = num >= den ? 1.0 : num / den;
            s = 1.0 - t;
        } else {
            t = 0.0;
            s = q1 <= 0.0 ? 1.0 : (b0 >= 0.0 ? 0.0 : -b0 / a00);
        }
    } else { /* region 1 */
        const double num = a11 + b1 - a01 - b0;
        if (num <= 0.0) {
            s = 0.0;
        } else {
            const double den = a00 - 2.0 * a01 + a11;
            s = num >= den ? 1.0 : num / den;
        }
        t = 1.0 - s;
    }
    return witness(p, add(add(tr->v0, scl(e0, s)), scl(e1, t)));
}

/* kernels.cpp:233-252: Cramer solve of u*e0 + v*e1 - t*d = -w */
typedef struct {
    int ok;
    double t, u, v;
} pierce_t;

static inline pierce_t pierce(v3 e0, v3 e1, v3 d, v3 w) {
    pierce_t r = {0, 0.0, 0.0, 0.0};
    const v3 pv = crs(d, e1);
    const double den = dot3(pv, e0);
    const double scale = len(d) * len(e0) * len(e1);
    if (fabs(den) <= PIERCE_EPS * scale) return r;
    const double inv = 1.0 / den;
    const v3 qv = crs(w, e0);
    r.t = dot3(qv, e1) * inv;
    r.u = dot3(pv, w) * inv;
    r.v = dot3(qv, d) * inv;
    r.ok = 1;
    return r;
}

/* kernels.cpp:256-316 */
static res_t seg_tri(v3 p0, v3 p1, const tri_t* tr) {
    if (same(p0, p1)) return pt_tri(p0, tr);
    const v3 d = sub(p1, p0), e0 = sub(tr->v1, tr->v0), e1 = sub(tr->v2, tr->v0);
    if (!tri_degenerate(tr)) {
        const pierce_t x = pierce(e0, e1, d, sub(p0, tr->v0));
        if (x.ok && x.u >= 0.0 && x.v >= 0.0 && x.u + x.v <= 1.0 && x.t >= 0.0 && x.t <= 1.0)
            return witness(add(p0, scl(d, x.t)), add(add(tr->v0, scl(e0, x.u)), scl(e1, x.v)));
    }
    res_t best;
    best.d = INFINITY;
    best.a = best.b = mk(0.0, 0.0, 0.0);
    const v3 ends[3][2] = {{tr->v0, tr->v1}, {tr->v0, tr->v2}, {tr->v1, tr->v2}};
    for (int k = 0; k < 3; ++k) {
        res_t c = seg_seg(p0, p1, ends[k][0], ends[k][1]);
        if (c.d < best.d) best = c;
    }
    res_t c = pt_tri(p0, tr);
    if (c.d < best.d) best = c;
    c = pt_tri(p1, tr);
    if (c.d < best.d) best = c;
    return best;
}

/* kernels.cpp:318-336 */
static int seg_tri_hit(v3 p0, v3 p1, const tri_t* tr) {
    const pierce_t x = pierce(sub(tr->v1, tr->v0), sub(tr->v2, tr->v0), sub(p1, p0), sub(p0, tr->v0));
    if (!x.ok) return 0;
    if (x.t < -BARY_SLACK || x.t > 1.0 + BARY_SLACK) return 0;
    if (x.u < -BARY_SLACK || x.v < -BARY_SLACK || x.u + x.v > 1.0 + BARY_SLACK) return 0;
    return 1;
}

static void put(const res_t* r, or_dist* o) {
    o->d = r->d;
    o->on_a[0] = r->a.x, o->on_a[1] = r->a.y, o->on_a[2] = r->a.z;
    o->on_b[0] = r->b.x, o->on_b[1] = r->b.y, o->on_b[2] = r->b.z;
}

void or_segment_segment_distance(const double* s6, const double* t6, or_dist* out) {
    res_t r = seg_seg(ld3(s6), ld3(s6 + 3), ld3(t6), ld3(t6 + 3));
    put(&r, out);
}
void or_point_triangle_distance(const double* p3, const double* t9, or_dist* out) {
    tri_t t = ld_tri(t9);
    res_t r = pt_tri(ld3(p3), &t);
    put(&r, out);
}
void or_segment_triangle_distance(const double* s6, const double* t9, or_dist* out) {
    tri_t t = ld_tri(t9);
    res_t r = seg_tri(ld3(s6), ld3(s6 + 3), &t);
    put(&r, out);
}
int or_segment_triangle_intersect(const double* s6, const double* t9) {
    tri_t t = ld_tri(t9);
    return seg_tri_hit(ld3(s6), ld3(s6 + 3), &t);
}
int or_triangle_is_degenerate(const double* t9) {
    tri_t t = ld_tri(t9);
    return tri_degenerate(&t);
}

/* ---- A17: the triangle-pair composition ---------------------------------
 * distance = min over the three directed edges of a (v0v1, v1v2, v2v0)
 * against b, then the three of b against a; first strict minimum wins.
 * Either triangle degenerate => +inf / no hit. */
static res_t tri_tri(const tri_t* a, const tri_t* b) {
    res_t best;
    best.d = INFINITY;
    best.a = best.b = mk(0.0, 0.0, 0.0);
    if (tri_degenerate(a) || tri_degenerate(b)) return best;
    const v3 ea[3][2] = {{a->v0, a->v1}, {a->v1, a->v2}, {a->v2, a->v0}};
    const v3 eb[3][2] = {{b->v0, b->v1}, {b->v1, b->v2}, {b->v2, b->v0}};
    for (int k = 0; k < 3; ++k) {
        res_t c = seg_tri(ea[k][0], ea[k][1], b);
        if (c.d < best.d) best = c;
    }
    for (int k = 0; k < 3; ++k) {
        res_t c = seg_tri(eb[k][0], eb[k][1], a);
        if (c.d < best.d) {
            best.d = c.d;
            best.a = c.b; /* the query segment lies on b here */
            best.b = c.a;
        }
    }
    return best;
}

static int tri_tri_hit(const tri_t* a, const tri_t* b) {
    if (tri_degenerate(a) || tri_degenerate(b)) return 0;
    if (seg_tri_hit(a->v0, a->v1, b) || seg_tri_hit(a->v1, a->v2, b) || seg_tri_hit(a->v2, a->v0, b))
        return 1;
    return seg_tri_hit(b->v0, b->v1, a) || seg_tri_hit(b->v1, b->v2, a) || seg_tri_hit(b->v2, b->v0, a);
}

void or_tri_tri_distance(const double* a9, const double* b9, or_dist* out) {
    tri_t a = ld_tri(a9), b = ld_tri(b9);
    res_t r = tri_tri(&a, &b);
    put(&r, out);
}
int or_tri_tri_intersects(const double* a9, const double* b9) {
    tri_t a = ld_tri(a9), b = ld_tri(b9);
    return tri_tri_hit(&a, &b);
}
void or_pairs_distance(const double* a9, const double* b9, uint64_t n, double* dist) {
    for (uint64_t k = 0; k < n; ++k) {
        tri_t a = ld_tri(a9 + 9 * k), b = ld_tri(b9 + 9 * k);
        dist[k] = tri_tri(&a, &b).d;
    }
}
void or_pairs_intersects(const double* a9, const double* b9, uint64_t n, uint8_t* hit) {
    for (uint64_t k = 0; k < n; ++k) {
        tri_t a = ld_tri(a9 + 9 * k), b = ld_tri(b9 + 9 * k);
        hit[k] = (uint8_t)tri_tri_hit(&a, &b);
    }
}

/* ---- row-parallel drivers (the role of executor.hpp:50-83 for_each_chunk:
 * workers claim row indices from an atomic counter, per-row results are
 * merged afterwards in row order so the answer never depends on threads) -- */
typedef struct {
    res_t r;
    uint64_t p;
    int found;
} row_best;

typedef struct {
    const double *a9, *b9;
    uint64_t m, row_begin, row_stride, rows;
    atomic_uint_fast64_t next;
    row_best* best;       /* distance */
    atomic_uint_fast64_t hit_p; /* intersects */
} mm_job;

static void* mm_dist_worker(void* arg) {
    mm_job* J = (mm_job*)arg;
    for (;;) {
        uint64_t k = atomic_fetch_add(&J->next, 1);
        if (k >= J->rows) break;
        const uint64_t i = J->row_begin + k * J->row_stride;
        const tri_t a = ld_tri(J->a9 + 9 * i);
        row_best rb;
        rb.found = 0;
        rb.p = 0;
        rb.r.d = INFINITY;
        for (uint64_t j = 0; j < J->m; ++j) {
            const tri_t b = ld_tri(J->b9 + 9 * j);
            res_t c = tri_tri(&a, &b);
            if (c.d < rb.r.d) {
                rb.r = c;
                rb.p = i * J->m + j;
                rb.found = 1;
            }
        }
        J->best[k] = rb;
    }
    return NULL;
}

static void* mm_hit_worker(void* arg) {
    mm_job* J = (mm_job*)arg;
    for (;;) {
        uint64_t k = atomic_fetch_add(&J->next, 1);
        if (k >= J->rows) break;
        const uint64_t i = J->row_begin + k * J->row_stride;
        if (i * J->m > atomic_load(&J->hit_p)) continue; /* cannot lower the answer */
        const tri_t a = ld_tri(J->a9 + 9 * i);
        for (uint64_t j = 0; j < J->m; ++j) {
            const tri_t b = ld_tri(J->b9 + 9 * j);
            if (tri_tri_hit(&a, &b)) {
                uint64_t p = i * J->m + j, seen = atomic_load(&J->hit_p);
                while (p < seen && !atomic_compare_exchange_weak(&J->hit_p, &seen, p)) {
                }
                break;
            }
        }
    }
    return NULL;
}

static void run_pool(int threads, void* (*fn)(void*), void* arg) {
    if (threads < 1) threads = 1;
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
    int started = 0;
    for (int w = 1; w < threads; ++w)
        if (pthread_create(&th[started], NULL, fn, arg) == 0) ++started;
    fn(arg);
    for (int w = 0; w < started; ++w) pthread_join(th[w], NULL);
    free(th);
}

static uint64_t row_count(uint64_t n, uint64_t* begin, uint64_t* end, uint64_t* stride) {
    if (*stride == 0) *stride = 1;
    if (*end > n) *end = n;
    return *begin < *end ? (*end - *begin + *stride - 1) / *stride : 0;
}

int or_mesh_mesh_distance(const double* a9, uint64_t n, const double* b9, uint64_t m,
                          uint64_t row_begin, uint64_t row_end, uint64_t row_stride, int threads,
                          or_mesh_dist* out) {
    mm_job J;
    memset(&J, 0, sizeof J);
    J.a9 = a9, J.b9 = b9, J.m = m, J.row_begin = row_begin;
    J.rows = row_count(n, &row_begin, &row_end, &row_stride);
    J.row_stride = row_stride;
    atomic_init(&J.next, 0);
    J.best = (row_best*)calloc(J.rows ? J.rows : 1, sizeof(row_best));
    run_pool(threads, mm_dist_worker, &J);
    row_best win;
    win.found = 0;
    win.p = UINT64_MAX;
    win.r.d = INFINITY;
    win.r.a = win.r.b = mk(0.0, 0.0, 0.0);
    for (uint64_t k = 0; k < J.rows; ++k)
        if (J.best[k].found && J.best[k].r.d < win.r.d) win = J.best[k];
    free(J.best);
    out->d = win.r.d;
    out->pair = win.found ? win.p : UINT64_MAX;
    out->found = win.found;
    out->on_a[0] = win.r.a.x, out->on_a[1] = win.r.a.y, out->on_a[2] = win.r.a.z;
    out->on_b[0] = win.r.b.x, out->on_b[1] = win.r.b.y, out->on_b[2] = win.r.b.z;
    return win.found;
}

int or_mesh_mesh_intersects(const double* a9, uint64_t n, const double* b9, uint64_t m,
                            uint64_t row_begin, uint64_t row_end, uint64_t row_stride, int threads,
                            uint64_t* pair_out) {
    mm_job J;
    memset(&J, 0, sizeof J);
    J.a9 = a9, J.b9 = b9, J.m = m, J.row_begin = row_begin;
    J.rows = row_count(n, &row_begin, &row_end, &row_stride);
    J.row_stride = row_stride;
    atomic_init(&J.next, 0);
    atomic_init(&J.hit_p, UINT64_MAX);
    run_pool(threads, mm_hit_worker, &J);
    *pair_out = atomic_load(&J.hit_p);
    return *pair_out != UINT64_MAX;
}

/* ---- table: one result per record, record = first argument ------------- */
typedef struct {
    const double *t9, *q9;
    const uint64_t* off;
    uint64_t nobj, mq;
    int op; /* 0 distance, 1 intersects */
    atomic_uint_fast64_t next;
    double* dist;
    uint8_t* hit;
    uint64_t* pair;
} tb_job;

static void* tb_worker(void* arg) {
    tb_job* J = (tb_job*)arg;
    for (;;) {
        uint64_t r = atomic_fetch_add(&J->next, 1);
        if (r >= J->nobj) break;
        const uint64_t lo = J->off[r], hi = J->off[r + 1];
        double best = INFINITY;
        uint64_t bp = UINT64_MAX;
        int done = 0;
        for (uint64_t i = lo; i < hi && !done; ++i) {
            const tri_t a = ld_tri(J->t9 + 9 * i);
            for (uint64_t j = 0; j < J->mq; ++j) {
                const tri_t b = ld_tri(J->q9 + 9 * j);
                const uint64_t p = (i - lo) * J->mq + j;
                if (J->op == 0) {
                    const double d = tri_tri(&a, &b).d;
                    if (d < best) best = d, bp = p;
                } else if (tri_tri_hit(&a, &b)) {
                    bp = p;
                    done = 1;
                    break;
                }
            }
        }
        if (J->op == 0) {
            if (J->dist) J->dist[r] = best;
        } else if (J->hit) {
            J->hit[r] = (uint8_t)(bp != UINT64_MAX);
        }
        if (J->pair) J->pair[r] = bp;
    }
    return NULL;
}

static void table_run(int op, const double* table9, const uint64_t* offsets, uint64_t n_objects,
                      const double* query9, uint64_t mq, int threads, double* dist, uint8_t* hit,
                      uint64_t* pair) {
    tb_job J;
    memset(&J, 0, sizeof J);
    J.t9 = table9, J.q9 = query9, J.off = offsets, J.nobj = n_objects, J.mq = mq, J.op = op;
    J.dist = dist, J.hit = hit, J.pair = pair;
    atomic_init(&J.next, 0);
    run_pool(threads, tb_worker, &J);
}

void or_table_distance(const double* table9, const uint64_t* offsets, uint64_t n_objects,
                       const double* query9, uint64_t mq, int threads, double* dist,
                       uint64_t* pair) {
    table_run(0, table9, offsets, n_objects, query9, mq, threads, dist, NULL, pair);
}

void or_table_intersects(const double* table9, const uint64_t* offsets, uint64_t n_objects,
                         const double* query9, uint64_t mq, int threads, uint8_t* hit,
                         uint64_t* pair) {
    table_run(1, table9, offsets, n_objects, query9, mq, threads, NULL, hit, pair);
}

/* ---- segment / point x mesh (kernels.cpp:347-432) ------------------------ */
typedef struct {
    const double *q, *t9;
    uint64_t n, m;
    int kind; /* 0 segment distance, 1 point distance, 2 segment intersects */
    atomic_uint_fast64_t next;
    double* dist;
    uint8_t* hit;
    uint64_t* face;
} q_job;

static void* q_worker(void* arg) {
    q_job* J = (q_job*)arg;
    for (;;) {
        const uint64_t k = atomic_fetch_add(&J->next, 1);
        if (k >= J->n) break;
        if (J->kind == 2) { /* intersects_mesh: lowest hit face, no degenerate skip */
            const double* s = J->q + 6 * k;
            uint64_t f = UINT64_MAX;
            for (uint64_t i = 0; i < J->m; ++i) {
                const tri_t t = ld_tri(J->t9 + 9 * i);
                if (seg_tri_hit(ld3(s), ld3(s + 3), &t)) {
                    f = i;
                    break;
                }
            }
            J->hit[k] = (uint8_t)(f != UINT64_MAX);
            J->face[k] = f;
            continue;
        }
        /* reduce_min_over_faces: strict '<' keeps the lowest face index */
        v3 p0, p1;
        int point = J->kind == 1;
        if (point) {
            p0 = p1 = ld3(J->q + 3 * k);
        } else {
            p0 = ld3(J->q + 6 * k), p1 = ld3(J->q + 6 * k + 3);
            point = same(p0, p1); /* kernels.cpp:388: degenerate segment -> point */
        }
        double best = INFINITY;
        uint64_t f = UINT64_MAX;
        for (uint64_t i = 0; i < J->m; ++i) {
            const tri_t t = ld_tri(J->t9 + 9 * i);
            if (tri_degenerate(&t)) continue;
            const double d = point ? pt_tri(p0, &t).d : seg_tri(p0, p1, &t).d;
            if (d < best) best = d, f = i;
        }
        J->dist[k] = best;
        J->face[k] = f;
    }
    return NULL;
}

static void q_run(int kind, const double* q, uint64_t n, const double* t9, uint64_t m, int threads, double* dist,
                  uint8_t* hit, uint64_t* face) {
    q_job J;
    memset(&J, 0, sizeof J);
    J.q = q, J.t9 = t9, J.n = n, J.m = m, J.kind = kind, J.dist = dist, J.hit = hit, J.face = face;
    atomic_init(&J.next, 0);
    run_pool(threads, q_worker, &J);
}

void or_segments_mesh_distance(const double* s6, uint64_t n, const double* t9, uint64_t m, int threads,
                               double* dist, uint64_t* face) {
    q_run(0, s6, n, t9, m, threads, dist, NULL, face);
}
void or_points_mesh_distance(const double* p3, uint64_t n, const double* t9, uint64_t m, int threads,
                             double* dist, uint64_t* face) {
    q_run(1, p3, n, t9, m, threads, dist, NULL, face);
}
void or_segments_mesh_intersects(const double* s6, uint64_t n, const double* t9, uint64_t m, int threads,
                                 uint8_t* hit, uint64_t* face) {
    q_run(2, s6, n, t9, m, threads, NULL, hit, face);
}

/* ---- pruned exact oracles (full-size parity) -------- */
typedef struct {
    double lo[3], hi[3];
} box_t;

static box_t face_box(const double* t) {
    box_t b;
    for (int k = 0; k < 3; ++k) {
        b.lo[k] = fmin(t[k], fmin(t[3 + k], t[6 + k]));
        b.hi[k] = fmax(t[k], fmax(t[3 + k], t[6 + k]));
    }
    return b;
}

static double box_dist2(const box_t* a, const box_t* b) {
    double s = 0.0;
    for (int k = 0; k < 3; ++k) {
        double g = fmax(0.0, fmax(a->lo[k] - b->hi[k], b->lo[k] - a->hi[k]));
        s += g * g;
    }
    return s;
}

/* Faces binned by centroid into a uniform grid of ~n/cap cells; CSR order. */
typedef struct {
    uint64_t ncell;
    uint64_t* start; /* ncell + 1 */
    uint64_t* face;  /* n, face ids grouped by cell (ascending within a cell) */
    box_t* cbox;     /* tight box of each cell's faces */
    box_t* fbox;     /* per face */
} grid_t;

static void grid_build(const double* t9, uint64_t n, grid_t* g) {
    g->fbox = (box_t*)malloc(sizeof(box_t) * (n ? n : 1));
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (uint64_t i = 0; i < n; ++i) {
        g->fbox[i] = face_box(t9 + 9 * i);
        for (int k = 0; k < 3; ++k) {
            lo[k] = fmin(lo[k], g->fbox[i].lo[k]);
            hi[k] = fmax(hi[k], g->fbox[i].hi[k]);
        }
    }
    double ext[3], vol = 1.0;
    int dims = 0;
    for (int k = 0; k < 3; ++k) {
        ext[k] = n ? hi[k] - lo[k] : 0.0;
        if (ext[k] > 0.0) vol *= ext[k], ++dims;
    }
    const double target = (double)(n / 64 + 1);
    const double side = dims ? pow(vol / target, 1.0 / dims) : 1.0;
    uint64_t d[3];
    for (int k = 0; k < 3; ++k) {
        d[k] = ext[k] > 0.0 && side > 0.0 ? (uint64_t)ceil(ext[k] / side) : 1;
        if (d[k] < 1) d[k] = 1;
        if (d[k] > 512) d[k] = 512;
    }
    g->ncell = d[0] * d[1] * d[2];
    g->start = (uint64_t*)calloc(g->ncell + 1, sizeof(uint64_t));
    uint64_t* cell = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t c = 0;
        for (int k = 2; k >= 0; --k) {
            const double x = (t9[9 * i + k] + t9[9 * i + 3 + k] + t9[9 * i + 6 + k]) / 3.0;
            int64_t q = ext[k] > 0.0 ? (int64_t)((x - lo[k]) / ext[k] * (double)d[k]) : 0;
            if (q < 0) q = 0;
            if (q >= (int64_t)d[k]) q = (int64_t)d[k] - 1;
            c = c * d[k] + (uint64_t)q;
        }
        cell[i] = c;
        g->start[c + 1]++;
    }
    for (uint64_t c = 0; c < g->ncell; ++c) g->start[c + 1] += g->start[c];
    uint64_t* fill = (uint64_t*)malloc(sizeof(uint64_t) * (g->ncell + 1));
    memcpy(fill, g->start, sizeof(uint64_t) * (g->ncell + 1));
    g->face = (uint64_t*)malloc(sizeof(uint64_t) * (n ? n : 1));
    for (uint64_t i = 0; i < n; ++i) g->face[fill[cell[i]]++] = i;
    g->cbox = (box_t*)malloc(sizeof(box_t) * g->ncell);
    for (uint64_t c = 0; c < g->ncell; ++c) {
        box_t b = {{INFINITY, INFINITY, INFINITY}, {-INFINITY, -INFINITY, -INFINITY}};
        for (uint64_t s = g->start[c]; s < g->start[c + 1]; ++s) {
            const box_t* f = &g->fbox[g->face[s]];
            for (int k = 0; k < 3; ++k) {
                b.lo[k] = fmin(b.lo[k], f->lo[k]);
                b.hi[k] = fmax(b.hi[k], f->hi[k]);
            }
        }
        g->cbox[c] = b;
    }
    free(fill);
    free(cell);
}

static void grid_free(grid_t* g) {
    free(g->start);
    free(g->face);
    free(g->cbox);
    free(g->fbox);
}

typedef struct {
    const double *a9, *b9;
    uint64_t m;
    const grid_t *ga, *gb;
    double thr2;
    int op; /* 0 distance, 1 intersects */
    atomic_uint_fast64_t next;
    pthread_mutex_t mu;
    double best_d;
    uint64_t best_p;
    res_t best_r;
    int found;
} pr_job;

static void* pr_worker(void* arg) {
    pr_job* J = (pr_job*)arg;
    double bd = INFINITY;
    uint64_t bp = UINT64_MAX;
    res_t br;
    int found = 0;
    for (;;) {
        const uint64_t ca = atomic_fetch_add(&J->next, 1);
        if (ca >= J->ga->ncell) break;
        if (J->ga->start[ca] == J->ga->start[ca + 1]) continue;
        for (uint64_t cb = 0; cb < J->gb->ncell; ++cb) {
            if (J->gb->start[cb] == J->gb->start[cb + 1]) continue;
            if (box_dist2(&J->ga->cbox[ca], &J->gb->cbox[cb]) > J->thr2) continue;
            for (uint64_t s = J->ga->start[ca]; s < J->ga->start[ca + 1]; ++s) {
                const uint64_t i = J->ga->face[s];
                const tri_t a = ld_tri(J->a9 + 9 * i);
                for (uint64_t u = J->gb->start[cb]; u < J->gb->start[cb + 1]; ++u) {
                    const uint64_t j = J->gb->face[u];
                    if (box_dist2(&J->ga->fbox[i], &J->gb->fbox[j]) > J->thr2) continue;
                    const uint64_t p = i * J->m + j;
                    if (J->op == 1) {
                        if (p < bp) {
                            const tri_t b = ld_tri(J->b9 + 9 * j);
                            if (tri_tri_hit(&a, &b)) bp = p, found = 1;
                        }
                        continue;
                    }
                    const tri_t b = ld_tri(J->b9 + 9 * j);
                    const res_t r = tri_tri(&a, &b);
                    if (r.d < bd || (r.d == bd && p < bp)) {
                        bd = r.d, bp = p, br = r, found = 1;
                    }
                }
            }
        }
    }
    pthread_mutex_lock(&J->mu);
    if (found) {
        if (J->op == 1) {
            if (!J->found || bp < J->best_p) J->best_p = bp;
        } else if (!J->found || bd < J->best_d || (bd == J->best_d && bp < J->best_p)) {
            J->best_d = bd, J->best_p = bp, J->best_r = br;
        }
        J->found = 1;
    }
    pthread_mutex_unlock(&J->mu);
    return NULL;
}

static double scale_of(const grid_t* g) {
    double s = 0.0;
    for (uint64_t c = 0; c < g->ncell; ++c)
        for (int k = 0; k < 3; ++k)
            if (g->start[c] != g->start[c + 1]) s = fmax(s, fmax(fabs(g->cbox[c].lo[k]), fabs(g->cbox[c].hi[k])));
    return s;
}

static int pruned_run(int op, const double* a9, uint64_t n, const double* b9, uint64_t m, double ub,
                      int threads, pr_job* J) {
    grid_t ga, gb;
    grid_build(a9, n, &ga);
    grid_build(b9, m, &gb);
    const double margin = 1e-9 * (1.0 + fmax(scale_of(&ga), scale_of(&gb)));
    const double thr = ub + margin;
    memset(J, 0, sizeof *J);
    J->a9 = a9, J->b9 = b9, J->m = m, J->ga = &ga, J->gb = &gb, J->op = op;
    J->thr2 = thr * thr;
    J->best_d = INFINITY;
    J->best_p = UINT64_MAX;
    atomic_init(&J->next, 0);
    pthread_mutex_init(&J->mu, NULL);
    run_pool(threads, pr_worker, J);
    pthread_mutex_destroy(&J->mu);
    grid_free(&ga);
    grid_free(&gb);
    return J->found;
}

int or_mesh_mesh_distance_pruned(const double* a9, uint64_t n, const double* b9, uint64_t m, double ub,
                                 int threads, or_mesh_dist* out) {
    pr_job J;
    pruned_run(0, a9, n, b9, m, ub, threads, &J);
    const int ok = J.found && J.best_d <= ub;
    out->d = ok ? J.best_d : INFINITY;
    out->pair = ok ? J.best_p : UINT64_MAX;
    out->found = ok;
    out->on_a[0] = J.best_r.a.x, out->on_a[1] = J.best_r.a.y, out->on_a[2] = J.best_r.a.z;
    out->on_b[0] = J.best_r.b.x, out->on_b[1] = J.best_r.b.y, out->on_b[2] = J.best_r.b.z;
    if (!ok) memset(out->on_a, 0, sizeof out->on_a), memset(out->on_b, 0, sizeof out->on_b);
    return ok;
}

int or_mesh_mesh_intersects_pruned(const double* a9, uint64_t n, const double* b9, uint64_t m,
                                   int threads, uint64_t* pair_out) {
    pr_job J;
    pruned_run(1, a9, n, b9, m, 0.0, threads, &J);
    *pair_out = J.found ? J.best_p : UINT64_MAX;
    return J.found;
}

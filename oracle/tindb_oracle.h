/* TEST INFRASTRUCTURE ONLY — the CPU checker for the triangle-pair hot path.
 *
 * A plain-C restatement of the reference's FP64 primitives
 * (/root/reference/proj/src/kernels.cpp) and of the SURVEY.md 8(a) A17
 * triangle-pair composition built from them. Only tests/, the smoke check in
 * __graft_entry__.py and bench.py's cpu_baseline leg may load it; the product
 * (paper_1808_09571_b200/) never does.
 *
 * Pinned against the reference itself: tests/test_oracle.py compares every
 * entry point bit-for-bit with oracle/_ref/libtindb_ref.so (the unmodified
 * reference sources) and with the committed golden vectors in tests/golden/.
 *
 * Layouts: a triangle is 9 doubles (v0 xyz, v1 xyz, v2 xyz) — exactly the
 * reference's TriangleMesh AoS (geometry.hpp:60-98, sizeof(Triangle) == 72);
 * a segment is 6 doubles (p0 xyz, p1 xyz).
 */
#ifndef TINDB_ORACLE_H
#define TINDB_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    double d;       /* distance, +inf when nothing was evaluated */
    double on_a[3]; /* witness on the first argument */
    double on_b[3]; /* witness on the second argument */
} or_dist;

typedef struct {
    double d;
    uint64_t pair; /* i*|B| + j, UINT64_MAX when not found */
    int found;
    double on_a[3], on_b[3];
} or_mesh_dist;

/* primitives (kernels.cpp:72, :138, :256, :318; geometry.hpp:75) */
void or_segment_segment_distance(const double* s6, const double* t6, or_dist* out);
void or_point_triangle_distance(const double* p3, const double* t9, or_dist* out);
void or_segment_triangle_distance(const double* s6, const double* t9, or_dist* out);
int or_segment_triangle_intersect(const double* s6, const double* t9);
int or_triangle_is_degenerate(const double* t9);

/* triangle pair (A17) */
void or_tri_tri_distance(const double* a9, const double* b9, or_dist* out);
int or_tri_tri_intersects(const double* a9, const double* b9);
void or_pairs_distance(const double* a9, const double* b9, uint64_t n, double* dist);
void or_pairs_intersects(const double* a9, const double* b9, uint64_t n, uint8_t* hit);

/* mesh x mesh over rows [row_begin,row_end) step row_stride of A, threads>=1 */
int or_mesh_mesh_distance(const double* a9, uint64_t n, const double* b9, uint64_t m,
                          uint64_t row_begin, uint64_t row_end, uint64_t row_stride, int threads,
                          or_mesh_dist* out);
int or_mesh_mesh_intersects(const double* a9, uint64_t n, const double* b9, uint64_t m,
                            uint64_t row_begin, uint64_t row_end, uint64_t row_stride, int threads,
                            uint64_t* pair_out);

/* Pruned exact oracles for full-size configurations.
 * Distance: the lexicographic minimum (d, p) over every pair whose exact
 * composition distance is <= ub, found by evaluating A17 only on face pairs
 * whose AABB distance is <= ub (+ a 1e-9-relative margin; face AABB distance
 * <= true distance <= reference distance + ulps). Equals the full answer
 * whenever ub >= the true minimum; found = 0 when no pair is <= ub.
 * Intersects: the lowest hit p among face pairs whose AABBs overlap within
 * the same margin (a hit needs the triangles to touch within the reference's
 * 1e-12 slack). Uniform cell grids on both meshes prune cell pairs first. */
int or_mesh_mesh_distance_pruned(const double* a9, uint64_t n, const double* b9, uint64_t m, double ub,
                                 int threads, or_mesh_dist* out);
int or_mesh_mesh_intersects_pruned(const double* a9, uint64_t n, const double* b9, uint64_t m,
                                   int threads, uint64_t* pair_out);

/* Per-query segment / point x mesh (kernels.cpp:382-432 distance_to_mesh,
 * intersects_mesh): distance + lowest face index (degenerate faces skipped,
 * kernels.cpp:350-357; a zero-length segment is a point query, :388), and
 * the lowest hit face (no degenerate skip, :407-432). face = UINT64_MAX when
 * none. Query-parallel over `threads`. */
void or_segments_mesh_distance(const double* s6, uint64_t n, const double* t9, uint64_t m, int threads,
                               double* dist, uint64_t* face);
void or_points_mesh_distance(const double* p3, uint64_t n, const double* t9, uint64_t m, int threads,
                             double* dist, uint64_t* face);
void or_segments_mesh_intersects(const double* s6, uint64_t n, const double* t9, uint64_t m, int threads,
                                 uint8_t* hit, uint64_t* face);

/* table: per record r (faces offsets[r]..offsets[r+1]) vs the query mesh,
 * record as the first argument (batch.cpp:31 eval_distance(record, arg)). */
void or_table_distance(const double* table9, const uint64_t* offsets, uint64_t n_objects,
                       const double* query9, uint64_t mq, int threads, double* dist,
                       uint64_t* pair);
void or_table_intersects(const double* table9, const uint64_t* offsets, uint64_t n_objects,
                         const double* query9, uint64_t mq, int threads, uint8_t* hit,
                         uint64_t* pair);

#ifdef __cplusplus
}
#endif
#endif

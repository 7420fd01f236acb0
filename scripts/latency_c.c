/* Per-call latency of the C ABI itself (no Python): the serving path's small
 * calls, wall time per call after warm-up. Build and run on the GPU box:
 *   gcc -O2 -Iinclude scripts/latency_c.c -Lpaper_1808_09571_b200 -ltindb_b200 \
 *       -Wl,-rpath,$PWD/paper_1808_09571_b200 -o /tmp/latency_c && /tmp/latency_c */
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "tindb_b200.h"

static double now_us(void) {
    struct timespec t;
    clock_gettime(CLOCK_MONOTONIC, &t);
    return t.tv_sec * 1e6 + t.tv_nsec * 1e-3;
}

#define TIME(name, call)                                                              \
    do {                                                                              \
        for (int i = 0; i < 50; ++i) call;                                            \
        double t0 = now_us();                                                         \
        for (int i = 0; i < 2000; ++i) call;                                          \
        printf("{\"call\": \"%s\", \"us_per_call\": %.1f, \"api\": \"C\"}\n", name,    \
               (now_us() - t0) / 2000);                                               \
    } while (0)

int main(void) {
    if (tdb_init(0) != 0) { fprintf(stderr, "init: %s\n", tdb_last_error()); return 1; }
    uint64_t n = tdb_gen_unit_sphere(1000, NULL);
    double* s = malloc(n * 9 * sizeof(double));
    tdb_gen_unit_sphere(1000, s);
    double* t = malloc(n * 9 * sizeof(double));
    for (uint64_t i = 0; i < n * 9; ++i) t[i] = s[i] + (i % 3 == 0 ? 2.5 : 0.0);
    double one2[9];
    for (int k = 0; k < 9; ++k) one2[k] = s[k] + (k % 3 == 2 ? 3.0 : 0.0);
    tdb_mesh a, b, o1, o2;
    tdb_mesh_upload(s, n, &a);
    tdb_mesh_upload(t, n, &b);
    tdb_mesh_upload(s, 1, &o1);
    tdb_mesh_upload(one2, 1, &o2);
    tdb_dist_out d;
    tdb_hit_out h;
    double seg[6] = {0, 0, 2, 0, 0, 3.0}, pt[3] = {0.1, 0.2, 1.5}, qd;
    uint64_t qf;
    uint8_t qh;
    TIME("distance 1x1", tdb_mesh_mesh_distance(o1, o2, &d));
    TIME("intersects 1x1", tdb_mesh_mesh_intersects(o1, o2, &h));
    TIME("segment query 1 x 1280 faces", tdb_segments_mesh_distance(seg, 1, a, &qd, &qf));
    TIME("point query 1 x 1280 faces", tdb_points_mesh_distance(pt, 1, a, &qd, &qf));
    TIME("segment intersects 1 x 1280", tdb_segments_mesh_intersects(seg, 1, a, &qh, &qf));
    TIME("distance 1280x1280", tdb_mesh_mesh_distance(a, b, &d));
    return 0;
}

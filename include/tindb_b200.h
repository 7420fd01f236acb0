/* tindb_b200 — B200-native (sm_100a) triangle-pair ST_3DDistance /
 * ST_3DIntersects engine behind a plain C ABI.
 *
 * Drop-in boundary for the reference `tindb` operator API
 * (/root/reference/proj/include/tindb/{kernels,batch}.hpp). The reference has
 * no mesh x mesh operator: kernels::run_batch returns TypeMismatch for
 * Mesh x Mesh (batch.cpp:49 eval_distance, batch.cpp:62 eval_intersects) and
 * kernels::distance_to_mesh throws for a mesh query (kernels.cpp:395-405).
 * The entry points below are what those branches bind;
 * each cites the reference interface it extends or replaces.
 *
 * Conventions
 *  - Triangles are 9 doubles (v0 xyz, v1 xyz, v2 xyz), i.e. exactly
 *    tindb::TriangleMesh::triangles.data() (geometry.hpp:60-98, 72 B/face).
 *  - Pair index p = i * |B| + j, i indexing the first mesh (the record /
 *    `a`), j the second (the argument / `b`). Ties keep the lowest p
 *    (kernels.cpp:359,368-376); intersects reports the lowest hit p
 *    (kernels.cpp:407-432).
 *  - Degenerate triangles (norm2((v1-v0)x(v2-v0)) <= 1e-30, geometry.hpp:75)
 *    make a mesh x mesh pair contribute +inf to distance minima and never
 *    intersect. Point / segment queries follow the store's
 *    has_degenerate_faces flags (tdb_geom_set_has_degenerate_faces).
 *  - Every call returns 0 on success and a negative TDB_E* code otherwise;
 *    tdb_last_error() (thread-local) holds the message. No C++ exception
 *    crosses this boundary. There is no CPU fallback: without a usable
 *    sm_100 device every compute call fails with TDB_E_CUDA.
 *  - Calls are thread-safe (the reference server calls plan_and_execute from
 *    one thread per connection, pg_server.cpp:231,496); device work is
 *    serialised per device.
 */
#ifndef TINDB_B200_H
#define TINDB_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TDB_OK 0
#define TDB_E_ARG (-1)   /* bad argument (maps to std::invalid_argument) */
#define TDB_E_CUDA (-2)  /* CUDA / device failure (maps to std::runtime_error) */
#define TDB_E_NOMEM (-3) /* device allocation failed */
#define TDB_E_PARSE (-4) /* malformed WKT: tindb::WktParseError (wkt.hpp:13); last_error = its what() */

typedef struct tdb_geom_s* tdb_mesh;  /* device-resident triangle soup (1 object) */
typedef struct tdb_geom_s* tdb_table; /* many objects: CSR face offsets + AABB headers */

/* Result of a mesh x mesh distance; mirrors kernels::DistanceResult
 * (kernels.hpp:28-34) extended with the pair index. */
typedef struct {
    double distance;   /* +inf when no non-degenerate pair exists */
    uint64_t pair;     /* i*|b| + j, UINT64_MAX when not found */
    uint64_t i, j;     /* face indices in a and b */
    double on_a[3];    /* witness on a's face i */
    double on_b[3];    /* witness on b's face j */
    int32_t found;
    int32_t _pad;
} tdb_dist_out;

/* Result of a mesh x mesh intersects; mirrors kernels::IntersectionResult
 * (kernels.hpp:43-48) with the lowest hit pair. */
typedef struct {
    int32_t hit;
    int32_t _pad;
    uint64_t pair; /* lowest hit pair, UINT64_MAX when none */
    uint64_t i, j;
} tdb_hit_out;

/* Per-call device statistics of the last compute call on this thread. */
typedef struct {
    double ms_total;        /* whole call on the device (events); one-launch small calls: host time from launch to results */
    double ms_filter;       /* the roofline kernel (fast FP64 filter / cull) */
    double ms_verify;       /* exact re-evaluation of candidate pairs */
    uint64_t pairs;         /* triangle pairs covered by the call */
    uint64_t items;         /* (A-tile x B-chunk) work items launched */
    uint64_t items_flagged; /* items re-scanned by the exact pass */
    uint64_t candidates;    /* pairs evaluated with the exact composition */
    uint64_t exact_pairs;   /* intersects: pairs that reached the exact predicate */
    uint64_t kernels;       /* kernel launches in the call */
    uint64_t pairs_evaluated; /* pairs run through the per-pair filter (== pairs in FULL mode) */
    uint64_t near_degenerate; /* exact-pass pairs flagged near-degenerate (tdb_last_near_degenerate) */
    int32_t rounds;       /* exact-pass rounds (>= 1; > 1 when a band was widened) */
    int32_t _pad;
} tdb_stats;

enum { TDB_OP_DISTANCE = 1, TDB_OP_INTERSECTS = 2 }; /* kernels::BatchOp (batch.hpp:14) */

/* Execution mode. FULL evaluates every triangle pair with the FP64 filter
 * (the roofline path, "no spatial index"). CULL additionally
 * skips whole (A-tile, B-chunk) items whose AABB lower bound cannot beat the
 * running answer — same results, fewer pair tests. */
enum { TDB_MODE_FULL = 0, TDB_MODE_CULL = 1 };

/* ---- runtime (replaces ExecutorConfig / for_each_chunk, executor.hpp:20-83) */
int tdb_init(int device);             /* idempotent; binds this thread to `device` */
int tdb_set_stream(void* cuda_stream); /* thread-local launch stream (NULL = library stream) */
int tdb_set_mode(int mode);           /* thread-local TDB_MODE_* */
const char* tdb_last_error(void);
int tdb_last_stats(tdb_stats* out);
/* Near-degenerate pairs met by the exact pass of the last call on this thread
 * (SPEC north star: "near-degenerate pairs logged"): a pair whose triangle
 * (or segment/triangle) is within 1e3 ulps of degenerate or of parallel.
 * Writes up to `cap` (object, pair) entries — object = A object / table row /
 * query index, pair = i*|B|+j / face index — as 2*cap uint64 values, and the
 * total count (which may exceed the 1024 entries kept) to *count_out. */
int tdb_last_near_degenerate(uint64_t* obj_pair_out, uint64_t cap, uint64_t* count_out);
int tdb_device_count(void);

/* ---- device geometry store (replaces the CPU mesh store, store_types.hpp:14-32) */
int tdb_mesh_upload(const double* tri9, uint64_t n_tris, tdb_mesh* out);
/* tri9 holds all objects' faces back to back; face_offsets has n_objects+1
 * entries (CSR), face_offsets[0] == 0. */
int tdb_table_upload(const double* tri9, const uint64_t* face_offsets, uint64_t n_objects,
                     tdb_table* out);
/* ---- device geometry loader (replaces tindb::parse_wkt, wkt.hpp:35, and the
 * TriangleMesh it builds; load_wkt_file / load_csv_text's WKT column,
 * store.hpp:62-71). The text is parsed in HBM; coordinates are bit-identical
 * to std::from_chars (wkt.cpp:84-95); POLYHEDRALSURFACE patches are
 * fan-triangulated as wkt.cpp:134-138. A literal the reference rejects
 * returns TDB_E_PARSE with the reference's WktParseError what() in
 * tdb_last_error() and its byte position in *err_pos (relative to the
 * literal); POINT / LINESTRING literals are not meshes (TDB_E_PARSE, pos 0). */
int tdb_mesh_from_wkt(const char* text, uint64_t len, tdb_mesh* out, uint64_t* err_pos);
/* n_lit literals text[lit_off[i], lit_off[i+1]) -> one table object each;
 * *err_literal names the first rejected literal. */
int tdb_table_from_wkt(const char* text, const uint64_t* lit_off, uint64_t n_lit, tdb_table* out,
                       uint64_t* err_literal, uint64_t* err_pos);
/* The store's faces back as host AoS, 9 doubles per face in face order. */
int tdb_geom_download(tdb_mesh g, double* tri9_out);
/* Its CSR face offsets (n_objects + 1 entries). */
int tdb_geom_offsets(tdb_mesh g, uint64_t* off_out);
int tdb_geom_info(tdb_mesh g, uint64_t* n_tris, uint64_t* n_objects, uint64_t* n_degenerate,
                  double* aabb6);
/* The reference's TriangleMesh::has_degenerate_faces per object
 * (geometry.hpp:84-97): point / segment distance queries against an object
 * (distance_to_mesh, run_batch with a Point / Segment literal over a mesh
 * column) skip its degenerate faces only when its flag is set
 * (reduce_min_over_faces, kernels.cpp:350,357); otherwise they evaluate them
 * through the reference's degenerate fallbacks (kernels.cpp:127-134,151-156).
 * flags: n_objects bytes (NULL = all set). A new store has every flag set,
 * what refresh_degeneracy_flag() gives for meshes that have degenerate faces
 * (parse_wkt and the generators call it, wkt.cpp:170, dataset.cpp:110).
 * Mesh x mesh (A17) always skips degenerate faces; intersects never does
 * (intersects_mesh has no skip, kernels.cpp:407-432). */
int tdb_geom_set_has_degenerate_faces(tdb_mesh g, const uint8_t* flags, uint64_t n_objects);
/* The distance filter's shared candidates (built on first use,
 * or here): as the B side, totals over the store's 64-face feature blocks of
 * non-degenerate faces, distinct vertices and distinct edges; as the A side,
 * the totals of the distinct edges and vertices of its super-tiles (256
 * tiles of 128 faces); super_edges: the distinct edges per 8,192 faces (B's
 * edge lists when a call's chunk allows them). No
 * reference counterpart (instrumentation for the roofline accounting). */
int tdb_geom_feature_counts(tdb_mesh g, uint64_t* faces, uint64_t* vertices, uint64_t* edges,
                            uint64_t* tile_edges, uint64_t* tile_vertices, uint64_t* super_edges);
void tdb_mesh_free(tdb_mesh m);
void tdb_table_free(tdb_table t);

/* ---- mesh x mesh (new kernels:: entries beside kernels.hpp:59-106) ------- */
int tdb_mesh_mesh_distance(tdb_mesh a, tdb_mesh b, tdb_dist_out* out);
int tdb_mesh_mesh_intersects(tdb_mesh a, tdb_mesh b, tdb_hit_out* out);
/* Row shard [row_begin,row_end) of a (multi-GPU split of the A axis); pair
 * indices stay global. */
int tdb_mesh_mesh_distance_rows(tdb_mesh a, uint64_t row_begin, uint64_t row_end, tdb_mesh b,
                                tdb_dist_out* out);
int tdb_mesh_mesh_intersects_rows(tdb_mesh a, uint64_t row_begin, uint64_t row_end, tdb_mesh b,
                                  tdb_hit_out* out);

/* ---- whole-column batch: run_batch(op, records, literal) for Mesh x Mesh
 * (batch.hpp:49-51). One slot per record, in record order; record is the
 * first argument. Any output pointer may be NULL. Rows [obj_begin,obj_end)
 * select a shard of the table (multi-GPU row split); outputs are indexed
 * from obj_begin. */
int tdb_table_eval(int op, tdb_table records, tdb_mesh literal, double* dist_out,
                   uint8_t* hit_out, uint64_t* pair_out);
int tdb_table_eval_rows(int op, tdb_table records, uint64_t obj_begin, uint64_t obj_end,
                        tdb_mesh literal, double* dist_out, uint8_t* hit_out,
                        uint64_t* pair_out);

/* ---- segment / point x mesh: the paper's drill-hole workload.
 * One result per query, in query order: distance_to_mesh (kernels.hpp:68-78,
 * kernels.cpp:382-405: min over non-degenerate faces, lowest face index on
 * ties, a zero-length segment is a point query) and intersects_mesh
 * (kernels.hpp:80-84, kernels.cpp:407-432: lowest hit face). face_out =
 * UINT64_MAX when there is none. Queries are host arrays: segments are 6
 * doubles (p0 xyz, p1 xyz, geometry.hpp:46-54), points 3. */
typedef struct tdb_queries_s* tdb_queries; /* device-resident segment or point column */
enum { TDB_QUERY_SEGMENTS = 0, TDB_QUERY_POINTS = 1 };
int tdb_queries_upload(const double* q, uint64_t n, int kind, tdb_queries* out);
void tdb_queries_free(tdb_queries q);
int tdb_queries_mesh_distance(tdb_queries q, tdb_mesh mesh, double* dist_out, uint64_t* face_out);
int tdb_queries_mesh_intersects(tdb_queries q, tdb_mesh mesh, uint8_t* hit_out, uint64_t* face_out);
/* run_batch with a Segment / Point literal over a mesh column (batch.cpp:44-48
 * eval_distance Mesh x Segment|Point, :59 eval_intersects Mesh x Segment):
 * per record distance_to_mesh(literal, record) / intersects_mesh(literal,
 * record); literal = 6 doubles (TDB_QUERY_SEGMENTS) or 3 (TDB_QUERY_POINTS,
 * distance only). face_out = lowest (hit) face within the record. */
int tdb_literal_table_eval(int op, int literal_kind, const double* literal, tdb_table records, double* dist_out,
                           uint8_t* hit_out, uint64_t* face_out);
/* one-shot forms: upload the host queries, evaluate, free */
int tdb_segments_mesh_distance(const double* seg6, uint64_t n, tdb_mesh mesh, double* dist_out,
                               uint64_t* face_out);
int tdb_points_mesh_distance(const double* pt3, uint64_t n, tdb_mesh mesh, double* dist_out,
                             uint64_t* face_out);
int tdb_segments_mesh_intersects(const double* seg6, uint64_t n, tdb_mesh mesh, uint8_t* hit_out,
                                 uint64_t* face_out);
uint64_t tdb_gen_drills(uint64_t seed, uint64_t count, int style, double* out6); /* dataset.cpp:141 */
/* The reference's complete result for one query against one triangle: for
 * TDB_OP_DISTANCE segment_triangle_distance / point_triangle_distance
 * (kernels.cpp:138-316: distance, closest points, SurfaceParams t,u,v), for
 * TDB_OP_INTERSECTS segment_triangle_intersect (kernels.cpp:318-336: hit,
 * point, IntersectionParams t,u,v,w). distance_to_mesh / intersects_mesh
 * report exactly this for their winning face (kernels.cpp:382-432): the
 * shim asks the query path for the face, then this for its details. */
typedef struct {
    double distance;
    double on_query[3]; /* closest_on_a */
    double on_face[3];  /* closest_on_b */
    double t, u, v, w;  /* SurfaceParams (w = 0) / IntersectionParams */
    int32_t hit;
    int32_t _pad;
    double point[3];    /* intersects: seg.p0 + clamp01(t) * d */
} tdb_face_result;
int tdb_query_face_result(int op, int query_kind, const double* query, const double* tri9, tdb_face_result* out);

/* ---- ST_3DVolume: mesh_volume (kernels.hpp:64-70, kernels.cpp:27-46),
 * permissive policy, bit-identical to the reference for the same chunk_size
 * (0 = ExecutorConfig default 4096; the chunk tree fixes the summation order,
 * executor.hpp:20-49). */
int tdb_mesh_volume(tdb_mesh m, uint64_t chunk_size, double* volume_out);
/* run_batch(Volume, records) over a mesh column (batch.cpp:23-29): one
 * volume per object, each with its own chunk tree (volume_out: n_objects). */
int tdb_table_volume(tdb_table t, uint64_t chunk_size, double* volume_out);

/* ---- device group: one process driving several B200s (SURVEY.md 8(b)
 * "tdb_init(int n_gpus): NCCL comm + streams", 8(e)). One worker thread per
 * device, one NCCL communicator per device (ncclCommInitAll). Geometry is
 * replicated on every member; mesh x mesh splits a's rows into contiguous
 * tile-aligned ranges, a table splits its objects into contiguous ranges of
 * near-equal face count. The only exchange is an NCCL MIN all-reduce: the
 * distance (its int64 bits), then the pair among the members holding it
 * (lowest pair on ties); intersects: the lowest hit pair, with a shared
 * lowest-hit word in peer memory so a hit on one device stops the work on
 * the devices holding higher rows. Results are those of the single-device
 * calls. Group calls are serialised per group. */
typedef struct tdb_group_s* tdb_group;
typedef struct tdb_gmesh_s* tdb_gmesh; /* a mesh or table replicated on the group */
int tdb_group_create(int n_devices, const int* devices, tdb_group* out); /* devices NULL = 0..n-1 */
void tdb_group_free(tdb_group g);
int tdb_group_size(tdb_group g);
int tdb_group_mesh_upload(tdb_group g, const double* tri9, uint64_t n_tris, tdb_gmesh* out);
int tdb_group_table_upload(tdb_group g, const double* tri9, const uint64_t* face_offsets,
                           uint64_t n_objects, tdb_gmesh* out);
void tdb_gmesh_free(tdb_gmesh m);
int tdb_group_mesh_mesh_distance(tdb_group g, tdb_gmesh a, tdb_gmesh b, tdb_dist_out* out);
int tdb_group_mesh_mesh_intersects(tdb_group g, tdb_gmesh a, tdb_gmesh b, tdb_hit_out* out);
/* run_batch(op, records, literal) with the records split over the group;
 * outputs as tdb_table_eval (one slot per record, record order). */
int tdb_group_table_eval(tdb_group g, int op, tdb_gmesh records, tdb_gmesh literal,
                         double* dist_out, uint8_t* hit_out, uint64_t* pair_out);
/* tdb_stats of member `member`'s share of the last group call */
int tdb_group_last_stats(tdb_group g, int member, tdb_stats* out);

/* ---- one-shot host-buffer entry points (upload + evaluate + free) -------- */
int tdb_distance_host(const double* a9, uint64_t n, const double* b9, uint64_t m,
                      tdb_dist_out* out);
int tdb_intersects_host(const double* a9, uint64_t n, const double* b9, uint64_t m,
                        tdb_hit_out* out);

/* ---- triangle-pair batch (parity / golden vectors): out[k] for (a[k], b[k]) */
int tdb_pairs_distance(const double* a9, const double* b9, uint64_t n, double* dist_out);
int tdb_pairs_intersects(const double* a9, const double* b9, uint64_t n, uint8_t* hit_out);

/* Filter value d~^2 of the FP64 roofline path for aligned pairs (testing the
 * filter's error bound against the exact composition). */
int tdb_pairs_filter(const double* a9, const double* b9, uint64_t n, double* d2_out);
/* The candidate set FULL mode evaluates (FP64 vertex/face and piercing, FP32
 * edge/edge relative to b's box centre o, as edge32_kernel does): d~^2 per
 * pair, and o (3) and the half-diagonal rB of b's box in origin_rb_out[4]
 * (testing eta_f32). */
int tdb_pairs_filter_f32(const double* a9, const double* b9, uint64_t n, double* d2_out, double* origin_rb_out);

/* ---- mesh generators ("mesh/geometry loader"; dataset.cpp:85-139). Return
 * the face count; write faces when out != NULL. Bit-identical to the
 * reference generator. */
uint64_t tdb_gen_unit_sphere(uint64_t face_target, double* out);
uint64_t tdb_gen_ore_body(uint64_t face_target, double* out);
/* NEW (not in the reference): nx*ny*2 CCW-up triangles over x,y in [0,1000],
 * z = U(-amp, amp) per lattice vertex from mt19937_64(seed) (rng.hpp:12-30). */
uint64_t tdb_gen_terrain(uint32_t nx, uint32_t ny, double amp, uint64_t seed, double* out);

/* ---- measurement helper: FP64 DFMA issue-rate microbenchmark (TFLOP/s) */
int tdb_fp64_peak(double* tflops_out, double* ms_out);

#ifdef __cplusplus
}
#endif
#endif /* TINDB_B200_H */

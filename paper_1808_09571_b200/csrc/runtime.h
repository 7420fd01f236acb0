// Host runtime internals: geometry handles, per-thread call context, errors.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <limits>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "exact.cuh"
#include "fast_pair.cuh"
#include "tdb_internal.h"
#include "tindb_b200.h"

namespace tdb {

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define CK(expr)                                                                              \
    do {                                                                                      \
        cudaError_t e_ = (expr);                                                              \
        if (e_ != cudaSuccess)                                                                \
            throw ::tdb::CudaError(std::string(#expr) + ": " + cudaGetErrorString(e_) + " (" + \
                                   __FILE__ + ":" + std::to_string(__LINE__) + ")");          \
    } while (0)

// A rejected WKT literal: the reference's WktParseError (wkt.hpp:13-23)
// what() and position, plus the literal's index in a multi-literal load.
struct WktError : std::invalid_argument {
    uint64_t literal, position;
    WktError(const std::string& what, uint64_t lit, uint64_t pos)
        : std::invalid_argument(what), literal(lit), position(pos) {}
};

inline double pos_inf_h() { return std::numeric_limits<double>::infinity(); }

struct Geom {
    int device = 0;
    uint64_t n = 0, n_pad = 0, n_obj = 0, n_degenerate = 0, n_chunks = 0;
    double* planes = nullptr;          // NF x n_pad
    uint64_t* d_off = nullptr;         // n_obj + 1
    Tile* d_tiles = nullptr;
    double* d_obj_stats = nullptr;     // n_obj x kObjStats
    double* d_tile_aabb = nullptr;     // per A tile: lo xyz, hi xyz
    std::vector<uint64_t> h_off;
    std::vector<Tile> h_tiles;
    std::vector<uint64_t> obj_tile0;   // first tile of each object (n_obj + 1)
    double stats[kObjStats] = {};      // aggregate: aabb lo/hi, max edge, max |coord|
    // FP32 copies of the vertices relative to `origin` (the first vertex of
    // face 0): 3 planes (one per vertex) of n_pad float4 (x, y, z, 0), for
    // the intersects FP32 pre-cull
    double origin[3] = {0.0, 0.0, 0.0};
    float* fplanes = nullptr;
    // per object: 1 = point / segment queries evaluate its degenerate faces
    // (TriangleMesh::has_degenerate_faces == false, kernels.cpp:350,357);
    // 0 (default) = skip them. tdb_geom_set_has_degenerate_faces.
    uint8_t* d_keep_deg = nullptr;
    std::vector<uint8_t> h_keep_deg;
    // feature blocks (tdb_internal.h kFB): built on first use as the B side
    // of a distance filter (geom_feature_blocks), kept until release
    mutable double* fblocks = nullptr;  // n_fblocks x kFBCap doubles
    mutable uint4* d_fhdr = nullptr;    // per block: faces, vertices, edges, doubles used
    mutable double4* d_fsph = nullptr;  // per block: bounding sphere of its live vertices (x, y, z, r)
    mutable uint64_t n_fblocks = 0;
    mutable uint32_t fblock_max = 0;    // max doubles used by one block
    mutable uint32_t fblock_max_pfv = 0;  //   ... by its face planes, face vertices and vertices
    mutable uint32_t fblock_max_e = 0;  //   ... by its edges
    mutable uint32_t fblock_max_f = 0;  //   ... by its faces
    // A side (tdb_internal.h kAER, kAVR): built on first use as the A side of
    // a distance filter (geom_edge_tiles)
    mutable double* aedges = nullptr;        // super-tiles' distinct edges, ordered by first tile
    mutable double* averts = nullptr;        // super-tiles' distinct vertices, ordered by first tile
    mutable std::vector<uint32_t> h_tile_st; // tile -> super-tile
    mutable std::vector<uint64_t> h_st_tile0;  // super-tile -> its first tile
    mutable std::vector<uint64_t> h_tile_eoff, h_tile_voff;  // n_tiles + 1: first entry with that first tile
    mutable std::vector<uint32_t> h_st_espan, h_st_vspan;    // per super-tile: max (second - first tile)
    mutable bool atiles_built = false;
    // B side: distinct edges per kBSuper faces (geom_super_bedges), as FP32
    // records (tdb_internal.h kBER) relative to bse_org = B's box centre;
    // bse_rB = the box's half-diagonal (bounds |P - bse_org|, eta_f32)
    mutable float4* bedges = nullptr;
    mutable double bse_org[3] = {0.0, 0.0, 0.0};
    mutable double bse_rB = 0.0;
    mutable std::vector<uint64_t> h_bseoff;  // per group of kBSuper faces: first entry
    mutable uint64_t* d_bseoff = nullptr;     // device copy
    // intersects (as B): bounding sphere of each kHitGroup faces (geom_hit_spheres)
    mutable double4* d_hsph = nullptr;
    std::shared_ptr<std::mutex> fmu = std::make_shared<std::mutex>();
};

// Builds g's feature blocks / edge tiles once (thread-safe; complete on the
// device when these return).
void geom_feature_blocks(const Geom& g, cudaStream_t st);
void geom_edge_tiles(const Geom& g, cudaStream_t st);
// atiles.cu: the super-tile edge and vertex lists (caller holds g.fmu)
void geom_super_tiles(const Geom& g, cudaStream_t st);
void geom_super_bedges(const Geom& g, cudaStream_t st);
// B's super-block edge lists, once (thread-safe)
void geom_bedges(const Geom& g, cudaStream_t st);
// B's per-kHitGroup-faces bounding spheres for the intersects block cull, once
void geom_hit_spheres(const Geom& g, cudaStream_t st);

// tri9: 9 doubles per face (AoS), on the host unless tri9_on_device
void geom_build(Geom* g, const double* tri9, uint64_t n, const uint64_t* host_off, uint64_t n_obj,
                cudaStream_t st, bool tri9_on_device = false);
void geom_release(Geom* g, cudaStream_t st);
// capi.cu: the calling thread's launch stream (binding its device), and
// "set tdb_last_error() and return rc" for code outside capi.cu (group.cu)
cudaStream_t call_stream();
void set_shared_hit(unsigned long long* p);  // this thread's Ctx::shared_hit
int set_error(int rc, const std::string& msg);
// Caller buffers <-> device (host_copy.cu): large pageable buffers go through
// pinned staging, page-locked ones straight to the copy engine. h2d is
// stream-ordered; the source must stay valid until the stream has passed the
// copy (every C-ABI call synchronises before it returns). d2h returns with
// the data in dst.
void h2d(void* dst, const void* src, size_t n, cudaStream_t st);
void d2h(void* dst, const void* src, size_t n, cudaStream_t st);
// WKT literals text[lit_off[i], lit_off[i+1]) (TIN Z / POLYHEDRALSURFACE Z),
// parsed on the device into g, one object per literal (csrc/wkt.cu).
void wkt_build(Geom* g, const char* text, const uint64_t* lit_off, uint64_t n_lit, cudaStream_t st);
// g's faces back to host AoS (9 doubles per face).
void geom_download(const Geom& g, double* host_tri9, cudaStream_t st);
// AABBs (lo xyz, hi xyz) of the uniform face chunks [c*len, (c+1)*len) of g.
void chunk_aabbs(const Geom& g, uint64_t len, double* out, cudaStream_t st);

// Near-degenerate log of the last call (host side, per thread).
struct NearHost {
    uint64_t count = 0;
    std::vector<uint64_t> entries;  // (object, pair) pairs, at most kNearLogCap
};

// Per-call execution context.
struct Ctx {
    cudaStream_t stream;
    int mode;
    int sms;
    tdb_stats* stats;
    NearHost* near;
    // device groups (group.cu): a lowest-hit word shared by every member
    // (peer memory over NVLink), so a hit on one device stops the others
    // early; null outside group calls
    unsigned long long* shared_hit = nullptr;
};

// Per-thread timing events, created once (cudaEventCreate per call costs
// more than a small call's kernels, and nothing leaks on an error path).
// A compute call records into e[0..3] and reads them before returning.
struct EventPair {
    cudaEvent_t e[4];
    EventPair() {
        for (auto& x : e) CK(cudaEventCreate(&x));
    }
    ~EventPair() {
        for (auto& x : e) cudaEventDestroy(x);
    }
};

// Events belong to a device: one set per (thread, current device).
inline EventPair& thread_events() {
    thread_local std::vector<std::unique_ptr<EventPair>> per_device;
    int dev = 0;
    CK(cudaGetDevice(&dev));
    if ((int)per_device.size() <= dev) per_device.resize(dev + 1);
    if (!per_device[dev]) per_device[dev] = std::make_unique<EventPair>();
    return *per_device[dev];
}

// Device side of the near-degenerate log for one call.
struct NearDev {
    NearLog log{nullptr, nullptr};
    cudaStream_t stream = nullptr;
    NearDev() = default;
    NearDev(const NearDev&) = delete;
    NearDev& operator=(const NearDev&) = delete;
    ~NearDev() {  // error paths: release without throwing
        if (log.count) cudaFreeAsync(log.count, stream);
        if (log.entries) cudaFreeAsync(log.entries, stream);
    }
    void alloc(cudaStream_t st) {
        stream = st;
        CK(cudaMallocAsync(&log.count, sizeof(unsigned long long), st));
        CK(cudaMallocAsync(&log.entries, 2 * kNearLogCap * sizeof(unsigned long long), st));
        CK(cudaMemsetAsync(log.count, 0, sizeof(unsigned long long), st));
    }
    // after the call's final synchronize
    void fetch(cudaStream_t st, NearHost* h) {
        unsigned long long c = 0;
        CK(cudaMemcpyAsync(&c, log.count, sizeof c, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        h->count = c;
        h->entries.assign(2 * std::min<uint64_t>(c, kNearLogCap), 0);
        if (!h->entries.empty())
            CK(cudaMemcpyAsync(h->entries.data(), log.entries, h->entries.size() * sizeof(uint64_t),
                               cudaMemcpyDeviceToHost, st));
        CK(cudaFreeAsync(log.count, st));
        log.count = nullptr;
        CK(cudaFreeAsync(log.entries, st));
        log.entries = nullptr;
        CK(cudaStreamSynchronize(st));
    }
};

// A-side selection: tiles [tile0, tile1) of A, rows restricted to
// [row_lo, row_hi); objects [obj0, obj1) (results indexed obj - obj0).
struct ASel {
    const Geom* A;
    uint64_t tile0, tile1, row_lo, row_hi, obj0, obj1;
};

// B-chunk length: halve from kChunk (down to `floor`, the kernel's staged
// sub-tile) until a launch has `waves` CTAs per SM, so small problems still
// spread over every SM (latency of small calls, the serving path).
inline uint64_t pick_chunk(uint64_t a_units, uint64_t nB, int sms, int waves, uint64_t floor = kSB) {
    uint64_t chunk = kChunk;
    const uint64_t target = (uint64_t)sms * (uint64_t)waves;
    while (chunk > floor && a_units * ((nB + chunk - 1) / chunk) < target) chunk >>= 1;
    return chunk;
}

// Work items (A tile x B chunk) one launch may carry: the per-item arrays
// cost 16 B each (2^27 items = 2 GB), and grids stay below 2^31 blocks.
// Larger selections run as consecutive tile batches whose per-object answers
// are merged (lexicographic (distance, pair); lowest hit pair). The
// TDB_MAX_ITEMS environment variable lowers the cap (tests).
inline uint64_t max_items() {
    static const uint64_t cap = [] {
        const char* e = getenv("TDB_MAX_ITEMS");
        const unsigned long long v = e ? strtoull(e, nullptr, 10) : 0;
        return v ? (uint64_t)v : (uint64_t)1 << 27;
    }();
    return cap;
}

// The selection split into batches of at most max_tiles A tiles (objects may
// straddle two batches; obj0/obj1 narrowed to each batch's tiles).
inline std::vector<ASel> tile_batches(const ASel& sel, uint64_t max_tiles) {
    std::vector<ASel> out;
    for (uint64_t t = sel.tile0; t < sel.tile1; t += max_tiles) {
        ASel b = sel;
        b.tile0 = t;
        b.tile1 = std::min(sel.tile1, t + max_tiles);
        b.obj0 = sel.A->h_tiles[b.tile0].obj;
        b.obj1 = (uint64_t)sel.A->h_tiles[b.tile1 - 1].obj + 1;
        out.push_back(b);
    }
    return out;
}

// Distance over an A selection against mesh B. Outputs per object (host):
// dist (+inf when none), pair (UINT64_MAX when none); for a single object
// also the witness (on_a, on_b).
void run_distance(const Ctx& cx, const ASel& sel, const Geom& B, double* dist, uint64_t* pair,
                  double* witness6);
void run_intersects(const Ctx& cx, const ASel& sel, const Geom& B, uint8_t* hit, uint64_t* pair);
// Small calls in one launch each (direct.cu): the exact composition on every
// pair, no filter / band. Used for one-object selections of at most
// direct_pairs(op) pairs, and for at most kDirectQueries one-shot queries of
// at most direct_query_pairs() (query, face) pairs. The limits are the
// measured crossovers against the pipeline on one B200
// (scripts/direct_crossover.py: distance ~1e5 pairs, intersects ~4e5).
// TDB_DIRECT_PAIRS overrides every limit (0 = never; tests run both paths on
// the same inputs).
constexpr int kDirectQueries = 16;
inline uint64_t direct_limit(uint64_t dflt) {
    const char* e = getenv("TDB_DIRECT_PAIRS");
    return e ? (uint64_t)strtoull(e, nullptr, 10) : dflt;
}
inline uint64_t direct_pairs(int op) {
    static const uint64_t d = direct_limit(98304), h = direct_limit(262144);
    return op == TDB_OP_DISTANCE ? d : h;
}
inline uint64_t direct_query_pairs() {
    static const uint64_t v = direct_limit(1ull << 16);
    return v;
}
bool direct_eligible(const ASel& sel, const Geom& B, int op);
void run_distance_direct(const Ctx& cx, const ASel& sel, const Geom& B, double* dist, uint64_t* pair,
                         double* witness6);
void run_intersects_direct(const Ctx& cx, const ASel& sel, const Geom& B, uint8_t* hit, uint64_t* pair);
void run_queries_direct(const Ctx& cx, int op, const double* q, uint64_t n, int kind, const Geom& B, double* dist,
                        uint8_t* hit, uint64_t* face);

// Exact composition over aligned pair arrays (parity entry points).
void run_pairs(const Ctx& cx, const double* a9, const double* b9, uint64_t n, double* dist,
               uint8_t* hit);

// origin != nullptr: FULL mode's candidate set (FP32 edge/edge relative to
// origin); else the FP64 per-pair filter
void run_pairs_filter(const Ctx& cx, const Geom& A, const Geom& B, double* d2, const double* origin = nullptr);

double fp64_peak(const Ctx& cx, double* ms);

// A device-resident set of segment or point queries (SoA planes).
constexpr int kQuerySegments = 0, kQueryPoints = 1;
struct QuerySet {
    int device = 0;
    int kind = kQuerySegments;
    int width = 6;  // doubles per query
    uint64_t n = 0, pad = 0;
    double* planes = nullptr;  // width x pad
};
void queries_build(QuerySet* qs, const double* host_q, uint64_t n, int kind, cudaStream_t st);

// Queries against mesh B, per query: distance_to_mesh (op TDB_OP_DISTANCE:
// dist + lowest face) or intersects_mesh (TDB_OP_INTERSECTS, segments: hit +
// lowest hit face).
void run_queries(const Ctx& cx, int op, const QuerySet& qs, const Geom& B, double* dist, uint8_t* hit,
                 uint64_t* face);

// One segment / point literal (q1.n == 1) against every object of table B
// (run_batch with a Segment / Point argument over Mesh records): per object
// distance_to_mesh (dist + lowest face) or intersects_mesh (hit + lowest hit
// face); faces are object-relative.
// The reference's full per-face result of one query against one triangle.
void run_face_result(const Ctx& cx, int op, int point, const double* q, const double* tri9, tdb_face_result* out);
void run_literal_table(const Ctx& cx, int op, const QuerySet& q1, const Geom& B, double* dist, uint8_t* hit,
                       uint64_t* face);

// mesh_volume (kernels.cpp:27-46) with the reference's fixed chunk tree.
double run_volume(const Ctx& cx, const Geom& g, uint64_t chunk);
// ... for every object of a table (out: n_obj doubles)
void run_volume_table(const Ctx& cx, const Geom& g, uint64_t chunk, double* out);

}  // namespace tdb

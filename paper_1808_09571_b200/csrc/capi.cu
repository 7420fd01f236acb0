// The C ABI (include/tindb_b200.h): argument checking, error mapping,
// per-thread stream/mode/stats, and the dispatch into the device runtime.
//
// Error behaviour mirrors the reference: invalid arguments are reported the
// way kernels.cpp:403 throws std::invalid_argument (TDB_E_ARG); device
// failures map to std::runtime_error (TDB_E_CUDA); nothing throws across the
// boundary.
#include <cuda_runtime.h>

#include <cstring>
#include <mutex>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "runtime.h"
#include "tindb_b200.h"

struct tdb_geom_s {
    tdb::Geom g;
};

struct tdb_queries_s {
    tdb::QuerySet q;
};

namespace {

thread_local std::string t_err;
thread_local cudaStream_t t_stream = nullptr;
thread_local bool t_stream_set = false;
thread_local int t_mode = TDB_MODE_FULL;
thread_local int t_device = -1;
thread_local tdb_stats t_stats{};
thread_local tdb::NearHost t_near;
thread_local uint64_t t_wkt_literal = 0, t_wkt_pos = 0;
thread_local unsigned long long* t_shared_hit = nullptr;

std::mutex g_mu;
std::vector<cudaStream_t> g_streams;  // library stream per device (stream-ordered frees)
std::vector<int> g_sms;
// Per-device pool of call streams (SURVEY.md 8(b) threading): every C-ABI
// call runs on a stream of its own, taken from the pool when the call starts
// and returned (idle) when it ends, so calls from concurrent threads — the
// reference server runs plan_and_execute on one thread per connection,
// pg_server.cpp:231,496 — overlap on the device instead of queueing on one
// stream. A thread that set its own stream (tdb_set_stream) uses that.
std::vector<std::vector<cudaStream_t>> g_pool;
thread_local int t_depth = 0;  // nesting of guarded() on this thread

struct HeldStream {
    cudaStream_t s = nullptr;
    int dev = -1;
    bool scoped = false;  // taken inside a C-ABI call: returned when it ends
    void give_back() {
        if (!s) return;
        cudaSetDevice(dev);
        cudaStreamSynchronize(s);  // idle before anyone else gets it (error paths included)
        std::lock_guard<std::mutex> lk(g_mu);
        g_pool[dev].push_back(s);
        s = nullptr;
    }
    ~HeldStream() { give_back(); }
};
thread_local HeldStream t_held;

cudaStream_t pooled_stream(int dev) {
    if (t_held.s && t_held.dev == dev) return t_held.s;
    t_held.give_back();
    cudaStream_t s = nullptr;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if (!g_pool[dev].empty()) {
            s = g_pool[dev].back();
            g_pool[dev].pop_back();
        }
    }
    if (!s) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    t_held.s = s;
    t_held.dev = dev;
    t_held.scoped = t_depth > 0;
    return s;
}

int fail(int code, const std::string& msg) {
    t_err = msg;
    return code;
}

// a call-scoped pooled stream goes back to the pool when the outermost
// C-ABI call of this thread returns (every call has synchronized by then)
struct CallScope {
    CallScope() { ++t_depth; }
    ~CallScope() {
        if (--t_depth == 0 && t_held.scoped) t_held.give_back();
    }
};

template <class F>
int guarded(F&& f) {
    CallScope scope;
    try {
        f();
        t_err.clear();
        return TDB_OK;
    } catch (const tdb::WktError& e) {
        t_wkt_literal = e.literal;
        t_wkt_pos = e.position;
        return fail(TDB_E_PARSE, e.what());
    } catch (const std::invalid_argument& e) {
        return fail(TDB_E_ARG, e.what());
    } catch (const std::bad_alloc& e) {
        return fail(TDB_E_NOMEM, e.what());
    } catch (const tdb::CudaError& e) {
        const std::string m = e.what();
        return fail(m.find("out of memory") != std::string::npos ? TDB_E_NOMEM : TDB_E_CUDA, m);
    } catch (const std::exception& e) {
        return fail(TDB_E_CUDA, e.what());
    }
}

void ensure_device() {
    if (t_device >= 0) {
        CK(cudaSetDevice(t_device));
        return;
    }
    int dev = 0;
    CK(cudaGetDevice(&dev));
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    if (n <= 0) throw tdb::CudaError("no CUDA device");
    cudaDeviceProp prop{};
    CK(cudaGetDeviceProperties(&prop, dev));
    if (prop.major != 10) throw tdb::CudaError("tindb_b200 requires an sm_100 (B200) device, found sm_" +
                                               std::to_string(prop.major * 10 + prop.minor));
    std::lock_guard<std::mutex> lk(g_mu);
    if ((int)g_streams.size() < n) {
        g_streams.resize(n, nullptr);
        g_sms.resize(n, 0);
        g_pool.resize(n);
    }
    if (!g_streams[dev]) {
        CK(cudaStreamCreateWithFlags(&g_streams[dev], cudaStreamNonBlocking));
        g_sms[dev] = prop.multiProcessorCount;
        // keep per-call scratch (cudaMallocAsync) cached in the device pool
        // instead of returning it to the OS at every synchronize
        cudaMemPool_t pool;
        CK(cudaDeviceGetDefaultMemPool(&pool, dev));
        uint64_t keep = UINT64_MAX;
        CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
        // Reserve headroom once: stores rebuilt every call (the one-shot host
        // path: ~1.2 GB of planes, feature blocks and staging per C2 batch)
        // otherwise fragment a pool sized to the working set, and the pool
        // then unmaps and maps memory inside cudaMallocAsync (0.1-0.9 s
        // stalls). TDB_POOL_RESERVE_MB overrides (0 = none).
        const char* e = getenv("TDB_POOL_RESERVE_MB");
        const size_t mb = e ? (size_t)strtoull(e, nullptr, 10) : 8192;
        if (mb) {
            void* p = nullptr;
            if (cudaMallocAsync(&p, mb << 20, g_streams[dev]) == cudaSuccess) {
                cudaFreeAsync(p, g_streams[dev]);
                cudaStreamSynchronize(g_streams[dev]);
            } else {
                cudaGetLastError();  // not enough memory: go without the headroom
            }
        }
    }
    t_device = dev;
}

// The library's stream on `dev` (created by the first call on it): handle
// frees are stream-ordered there, back into the device pool.
cudaStream_t lib_stream(int dev) {
    std::lock_guard<std::mutex> lk(g_mu);
    return dev >= 0 && dev < (int)g_streams.size() ? g_streams[dev] : nullptr;
}

tdb::Ctx ctx() {
    ensure_device();
    tdb::Ctx c;
    c.stream = t_stream_set ? t_stream : pooled_stream(t_device);
    c.mode = t_mode;
    c.sms = g_sms[t_device];
    c.stats = &t_stats;
    t_near.count = 0;
    t_near.entries.clear();
    c.near = &t_near;
    c.shared_hit = t_shared_hit;
    return c;
}

void need(bool ok, const char* what) {
    if (!ok) throw std::invalid_argument(what);
}

tdb::ASel mesh_rows(const tdb::Geom& A, uint64_t r0, uint64_t r1) {
    need(A.n_obj == 1, "first argument must be a mesh (one object)");
    need(r0 <= r1 && r1 <= A.n, "row range out of bounds");
    tdb::ASel s;
    s.A = &A;
    s.tile0 = r0 / tdb::kTile;
    s.tile1 = (r1 + tdb::kTile - 1) / tdb::kTile;
    if (r0 == r1) s.tile1 = s.tile0;
    s.row_lo = r0;
    s.row_hi = r1;
    s.obj0 = 0;
    s.obj1 = 1;
    return s;
}

void fill_dist(tdb_dist_out* out, double d, uint64_t p, const double* w6, uint64_t m) {
    std::memset(out, 0, sizeof *out);
    out->distance = d;
    out->pair = p;
    out->found = p != ~0ull;
    out->i = out->found ? p / m : ~0ull;
    out->j = out->found ? p % m : ~0ull;
    if (w6) {
        std::memcpy(out->on_a, w6, 3 * sizeof(double));
        std::memcpy(out->on_b, w6 + 3, 3 * sizeof(double));
    }
}

void fill_hit(tdb_hit_out* out, uint64_t p, uint64_t m) {
    std::memset(out, 0, sizeof *out);
    out->pair = p;
    out->hit = p != ~0ull;
    out->i = out->hit ? p / m : ~0ull;
    out->j = out->hit ? p % m : ~0ull;
}

void upload(const double* tri9, uint64_t n, const uint64_t* off, uint64_t n_obj, tdb_geom_s** out) {
    need(out != nullptr, "null output handle");
    need(n == 0 || tri9 != nullptr, "null triangle array");
    need(off[0] == 0 && off[n_obj] == n, "face offsets must start at 0 and end at n_tris");
    for (uint64_t o = 0; o < n_obj; ++o) need(off[o] <= off[o + 1], "face offsets must be non-decreasing");
    tdb::Ctx c = ctx();
    auto* h = new tdb_geom_s();
    h->g.device = t_device;
    try {
        tdb::geom_build(&h->g, tri9, n, off, n_obj, c.stream);
    } catch (...) {
        tdb::geom_release(&h->g, c.stream);
        delete h;
        throw;
    }
    *out = h;
}

}  // namespace

cudaStream_t tdb::call_stream() { return ctx().stream; }

void tdb::set_shared_hit(unsigned long long* p) { t_shared_hit = p; }

int tdb::set_error(int rc, const std::string& msg) { return rc == TDB_OK ? (t_err.clear(), rc) : fail(rc, msg); }

extern "C" {

int tdb_init(int device) {
    return guarded([&] {
        int n = 0;
        CK(cudaGetDeviceCount(&n));
        need(device >= 0 && device < n, "device index out of range");
        CK(cudaSetDevice(device));
        t_device = -1;
        ensure_device();
    });
}

int tdb_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

int tdb_set_stream(void* s) {
    t_stream = static_cast<cudaStream_t>(s);
    t_stream_set = s != nullptr;
    return TDB_OK;
}

int tdb_set_mode(int mode) {
    if (mode != TDB_MODE_FULL && mode != TDB_MODE_CULL) return fail(TDB_E_ARG, "unknown mode");
    t_mode = mode;
    return TDB_OK;
}

const char* tdb_last_error(void) { return t_err.c_str(); }

int tdb_last_near_degenerate(uint64_t* obj_pair_out, uint64_t cap, uint64_t* count_out) {
    if (!count_out || (cap && !obj_pair_out)) return fail(TDB_E_ARG, "null output");
    *count_out = t_near.count;
    const uint64_t n = std::min<uint64_t>(cap, t_near.entries.size() / 2);
    if (n) std::memcpy(obj_pair_out, t_near.entries.data(), 2 * n * sizeof(uint64_t));
    return TDB_OK;
}

int tdb_last_stats(tdb_stats* out) {
    if (!out) return fail(TDB_E_ARG, "null stats");
    *out = t_stats;
    return TDB_OK;
}

int tdb_mesh_upload(const double* tri9, uint64_t n, tdb_mesh* out) {
    return guarded([&] {
        const uint64_t off[2] = {0, n};
        upload(tri9, n, off, 1, out);
    });
}

int tdb_table_upload(const double* tri9, const uint64_t* off, uint64_t n_obj, tdb_table* out) {
    return guarded([&] {
        need(off != nullptr, "null face offsets");
        upload(tri9, off[n_obj], off, n_obj, out);
    });
}

int tdb_mesh_from_wkt(const char* text, uint64_t len, tdb_mesh* out, uint64_t* err_pos) {
    const uint64_t off[2] = {0, len};
    return tdb_table_from_wkt(text, off, 1, out, nullptr, err_pos);
}

int tdb_table_from_wkt(const char* text, const uint64_t* lit_off, uint64_t n_lit, tdb_table* out,
                       uint64_t* err_literal, uint64_t* err_pos) {
    const int rc = guarded([&] {
        need(out != nullptr, "null output handle");
        need(lit_off != nullptr && (text != nullptr || lit_off[n_lit] == 0), "null WKT text or offsets");
        need(lit_off[0] == 0, "literal offsets must start at 0");
        tdb::Ctx c = ctx();
        auto* h = new tdb_geom_s();
        h->g.device = t_device;
        try {
            tdb::wkt_build(&h->g, text, lit_off, n_lit, c.stream);
        } catch (...) {
            tdb::geom_release(&h->g, c.stream);
            delete h;
            throw;
        }
        *out = h;
    });
    if (rc == TDB_E_PARSE) {
        if (err_literal) *err_literal = t_wkt_literal;
        if (err_pos) *err_pos = t_wkt_pos;
    }
    return rc;
}

int tdb_geom_offsets(tdb_mesh g, uint64_t* off_out) {
    return guarded([&] {
        need(g != nullptr && off_out != nullptr, "null argument");
        std::memcpy(off_out, g->g.h_off.data(), (g->g.n_obj + 1) * sizeof(uint64_t));
    });
}

int tdb_geom_download(tdb_mesh g, double* tri9_out) {
    return guarded([&] {
        need(g != nullptr, "null handle");
        need(tri9_out != nullptr || g->g.n == 0, "null output");
        tdb::geom_download(g->g, tri9_out, ctx().stream);
    });
}

int tdb_geom_info(tdb_mesh g, uint64_t* n, uint64_t* n_obj, uint64_t* n_deg, double* aabb6) {
    return guarded([&] {
        need(g != nullptr, "null handle");
        if (n) *n = g->g.n;
        if (n_obj) *n_obj = g->g.n_obj;
        if (n_deg) *n_deg = g->g.n_degenerate;
        if (aabb6) std::memcpy(aabb6, g->g.stats, 6 * sizeof(double));
    });
}

int tdb_geom_set_has_degenerate_faces(tdb_mesh g, const uint8_t* flags, uint64_t n_objects) {
    return guarded([&] {
        need(g != nullptr, "null handle");
        need(n_objects == g->g.n_obj, "n_objects must equal the store's object count");
        for (uint64_t o = 0; o < n_objects; ++o) g->g.h_keep_deg[o] = flags && !flags[o] ? 1 : 0;
        cudaSetDevice(g->g.device);
        const cudaStream_t st = lib_stream(g->g.device);
        if (n_objects) {
            CK(cudaMemcpyAsync(g->g.d_keep_deg, g->g.h_keep_deg.data(), n_objects, cudaMemcpyHostToDevice, st));
            CK(cudaStreamSynchronize(st));
        }
    });
}

int tdb_geom_feature_counts(tdb_mesh g, uint64_t* faces, uint64_t* vertices, uint64_t* edges,
                            uint64_t* tile_edges, uint64_t* tile_vertices, uint64_t* super_edges) {
    return guarded([&] {
        need(g != nullptr, "null handle");
        cudaSetDevice(g->g.device);
        const cudaStream_t st = lib_stream(g->g.device);
        tdb::geom_feature_blocks(g->g, st);
        std::vector<uint4> h(g->g.n_fblocks);
        if (!h.empty()) {
            CK(cudaMemcpyAsync(h.data(), g->g.d_fhdr, h.size() * sizeof(uint4), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
        }
        uint64_t t[3] = {0, 0, 0};
        for (const uint4& b : h) t[0] += b.x, t[1] += b.y, t[2] += b.z;
        if (faces) *faces = t[0];
        if (vertices) *vertices = t[1];
        if (edges) *edges = t[2];
        if (tile_edges || tile_vertices) {
            tdb::geom_edge_tiles(g->g, st);
            if (tile_edges) *tile_edges = g->g.h_tile_eoff.empty() ? 0 : g->g.h_tile_eoff.back();
            if (tile_vertices) *tile_vertices = g->g.h_tile_voff.empty() ? 0 : g->g.h_tile_voff.back();
        }
        if (super_edges) {
            tdb::geom_bedges(g->g, st);
            *super_edges = g->g.h_bseoff.empty() ? 0 : g->g.h_bseoff.back();
        }
    });
}

void tdb_mesh_free(tdb_mesh m) {
    if (!m) return;
    cudaSetDevice(m->g.device);
    const cudaStream_t st = lib_stream(m->g.device);
    tdb::geom_release(&m->g, st);
    // the frees complete now, so the device pool hands this memory to the
    // next allocation on any stream (without it, a store rebuilt every call
    // — the one-shot host path — grew the pool by its size, 0.3-0.9 s)
    cudaStreamSynchronize(st);
    delete m;
}

void tdb_table_free(tdb_table t) { tdb_mesh_free(t); }

int tdb_mesh_mesh_distance_rows(tdb_mesh a, uint64_t r0, uint64_t r1, tdb_mesh b, tdb_dist_out* out) {
    return guarded([&] {
        need(a && b && out, "null argument");
        need(b->g.n_obj == 1, "second argument must be a mesh (one object)");
        tdb::Ctx c = ctx();
        double d = 0, w[6];
        uint64_t p = 0;
        tdb::run_distance(c, mesh_rows(a->g, r0, r1), b->g, &d, &p, w);
        fill_dist(out, d, p, w, b->g.n);
    });
}

int tdb_mesh_mesh_distance(tdb_mesh a, tdb_mesh b, tdb_dist_out* out) {
    if (!a) return fail(TDB_E_ARG, "null argument");
    return tdb_mesh_mesh_distance_rows(a, 0, a->g.n, b, out);
}

int tdb_mesh_mesh_intersects_rows(tdb_mesh a, uint64_t r0, uint64_t r1, tdb_mesh b, tdb_hit_out* out) {
    return guarded([&] {
        need(a && b && out, "null argument");
        need(b->g.n_obj == 1, "second argument must be a mesh (one object)");
        tdb::Ctx c = ctx();
        uint64_t p = 0;
        uint8_t h = 0;
        tdb::run_intersects(c, mesh_rows(a->g, r0, r1), b->g, &h, &p);
        fill_hit(out, p, b->g.n);
    });
}

int tdb_mesh_mesh_intersects(tdb_mesh a, tdb_mesh b, tdb_hit_out* out) {
    if (!a) return fail(TDB_E_ARG, "null argument");
    return tdb_mesh_mesh_intersects_rows(a, 0, a->g.n, b, out);
}

int tdb_table_eval_rows(int op, tdb_table t, uint64_t o0, uint64_t o1, tdb_mesh lit, double* dist,
                        uint8_t* hit, uint64_t* pair) {
    return guarded([&] {
        need(t && lit, "null argument");
        need(op == TDB_OP_DISTANCE || op == TDB_OP_INTERSECTS, "unknown op");
        need(lit->g.n_obj == 1, "literal must be a mesh (one object)");
        need(o0 <= o1 && o1 <= t->g.n_obj, "object range out of bounds");
        tdb::Ctx c = ctx();
        const tdb::Geom& A = t->g;
        tdb::ASel s;
        s.A = &A;
        s.tile0 = A.obj_tile0[o0];
        s.tile1 = A.obj_tile0[o1];
        s.row_lo = A.h_off[o0];
        s.row_hi = A.h_off[o1];
        s.obj0 = o0;
        s.obj1 = o1;
        const uint64_t k = o1 - o0;
        std::vector<uint64_t> p(k);
        if (op == TDB_OP_DISTANCE) {
            std::vector<double> d(k);
            tdb::run_distance(c, s, lit->g, d.data(), p.data(), nullptr);
            if (dist) std::memcpy(dist, d.data(), k * sizeof(double));
        } else {
            std::vector<uint8_t> h(k);
            tdb::run_intersects(c, s, lit->g, h.data(), p.data());
            if (hit) std::memcpy(hit, h.data(), k);
        }
        if (pair) std::memcpy(pair, p.data(), k * sizeof(uint64_t));
    });
}

int tdb_table_eval(int op, tdb_table t, tdb_mesh lit, double* dist, uint8_t* hit, uint64_t* pair) {
    if (!t) return fail(TDB_E_ARG, "null argument");
    return tdb_table_eval_rows(op, t, 0, t->g.n_obj, lit, dist, hit, pair);
}

int tdb_distance_host(const double* a9, uint64_t n, const double* b9, uint64_t m, tdb_dist_out* out) {
    tdb_mesh a = nullptr, b = nullptr;
    int rc = tdb_mesh_upload(a9, n, &a);
    if (rc == TDB_OK) rc = tdb_mesh_upload(b9, m, &b);
    if (rc == TDB_OK) rc = tdb_mesh_mesh_distance(a, b, out);
    const std::string err = t_err;
    tdb_mesh_free(a);
    tdb_mesh_free(b);
    t_err = err;
    return rc;
}

int tdb_intersects_host(const double* a9, uint64_t n, const double* b9, uint64_t m, tdb_hit_out* out) {
    tdb_mesh a = nullptr, b = nullptr;
    int rc = tdb_mesh_upload(a9, n, &a);
    if (rc == TDB_OK) rc = tdb_mesh_upload(b9, m, &b);
    if (rc == TDB_OK) rc = tdb_mesh_mesh_intersects(a, b, out);
    const std::string err = t_err;
    tdb_mesh_free(a);
    tdb_mesh_free(b);
    t_err = err;
    return rc;
}

int tdb_pairs_distance(const double* a9, const double* b9, uint64_t n, double* dist) {
    return guarded([&] {
        need(n == 0 || (a9 && b9 && dist), "null argument");
        tdb::run_pairs(ctx(), a9, b9, n, dist, nullptr);
    });
}

int tdb_pairs_intersects(const double* a9, const double* b9, uint64_t n, uint8_t* hit) {
    return guarded([&] {
        need(n == 0 || (a9 && b9 && hit), "null argument");
        tdb::run_pairs(ctx(), a9, b9, n, nullptr, hit);
    });
}

int tdb_pairs_filter(const double* a9, const double* b9, uint64_t n, double* d2) {
    tdb_mesh a = nullptr, b = nullptr;
    int rc = tdb_mesh_upload(a9, n, &a);
    if (rc == TDB_OK) rc = tdb_mesh_upload(b9, n, &b);
    if (rc == TDB_OK)
        rc = guarded([&] { tdb::run_pairs_filter(ctx(), a->g, b->g, d2); });
    const std::string err = t_err;
    tdb_mesh_free(a);
    tdb_mesh_free(b);
    t_err = err;
    return rc;
}

int tdb_pairs_filter_f32(const double* a9, const double* b9, uint64_t n, double* d2, double* origin_rb) {
    tdb_mesh a = nullptr, b = nullptr;
    int rc = tdb_mesh_upload(a9, n, &a);
    if (rc == TDB_OK) rc = tdb_mesh_upload(b9, n, &b);
    if (rc == TDB_OK)
        rc = guarded([&] {
            need(origin_rb != nullptr, "null origin output");
            const double* s = b->g.stats;  // as geom_super_bedges: B's box centre and half-diagonal
            double r2 = 0.0;
            for (int k = 0; k < 3; ++k) {
                origin_rb[k] = 0.5 * (s[k] + s[3 + k]);
                r2 += (s[3 + k] - s[k]) * (s[3 + k] - s[k]);
            }
            origin_rb[3] = 0.5 * std::sqrt(r2) * (1.0 + 1e-12);
            tdb::run_pairs_filter(ctx(), a->g, b->g, d2, origin_rb);
        });
    const std::string err = t_err;
    tdb_mesh_free(a);
    tdb_mesh_free(b);
    t_err = err;
    return rc;
}

int tdb_query_face_result(int op, int kind, const double* q, const double* tri9, tdb_face_result* out) {
    return guarded([&] {
        need(q && tri9 && out, "null argument");
        need(op == TDB_OP_DISTANCE || op == TDB_OP_INTERSECTS, "unknown op");
        need(kind == TDB_QUERY_SEGMENTS || kind == TDB_QUERY_POINTS, "unknown query kind");
        need(!(op == TDB_OP_INTERSECTS && kind == TDB_QUERY_POINTS), "intersects takes a segment");
        tdb::run_face_result(ctx(), op, kind == TDB_QUERY_POINTS, q, tri9, out);
    });
}

int tdb_queries_upload(const double* q, uint64_t n, int kind, tdb_queries* out) {
    return guarded([&] {
        need(out != nullptr, "null output handle");
        need(n == 0 || q != nullptr, "null query array");
        need(kind == TDB_QUERY_SEGMENTS || kind == TDB_QUERY_POINTS, "unknown query kind");
        tdb::Ctx c = ctx();
        auto* h = new tdb_queries_s();
        h->q.device = t_device;
        try {
            tdb::queries_build(&h->q, q, n, kind == TDB_QUERY_SEGMENTS ? tdb::kQuerySegments : tdb::kQueryPoints,
                               c.stream);
        } catch (...) {
            cudaFreeAsync(h->q.planes, c.stream);
            delete h;
            throw;
        }
        *out = h;
    });
}

void tdb_queries_free(tdb_queries q) {
    if (!q) return;
    cudaSetDevice(q->q.device);
    cudaFreeAsync(q->q.planes, lib_stream(q->q.device));
    delete q;
}

int tdb_queries_mesh_distance(tdb_queries q, tdb_mesh mesh, double* dist_out, uint64_t* face_out) {
    return guarded([&] {
        need(q && mesh && (q->q.n == 0 || (dist_out && face_out)), "null argument");
        need(mesh->g.n_obj == 1, "the argument must be a mesh (one object)");
        tdb::run_queries(ctx(), TDB_OP_DISTANCE, q->q, mesh->g, dist_out, nullptr, face_out);
    });
}

int tdb_queries_mesh_intersects(tdb_queries q, tdb_mesh mesh, uint8_t* hit_out, uint64_t* face_out) {
    return guarded([&] {
        need(q && mesh && (q->q.n == 0 || (hit_out && face_out)), "null argument");
        need(q->q.kind == tdb::kQuerySegments, "intersects takes segment queries (intersects_mesh, kernels.hpp:80)");
        need(mesh->g.n_obj == 1, "the argument must be a mesh (one object)");
        tdb::run_queries(ctx(), TDB_OP_INTERSECTS, q->q, mesh->g, nullptr, hit_out, face_out);
    });
}

static int one_shot_queries(const double* q, uint64_t n, int kind, int op, tdb_mesh mesh, double* dist,
                            uint8_t* hit, uint64_t* face) {
    if (mesh && n > 0 && n <= (uint64_t)tdb::kDirectQueries && n * mesh->g.n <= tdb::direct_query_pairs())
        return guarded([&] {  // small call: one launch, no query upload (direct.cu)
            need(q != nullptr && face != nullptr && (op == TDB_OP_DISTANCE ? dist != nullptr : hit != nullptr),
                 "null argument");
            need(kind == TDB_QUERY_SEGMENTS || kind == TDB_QUERY_POINTS, "unknown query kind");
            need(op == TDB_OP_DISTANCE || kind == TDB_QUERY_SEGMENTS,
                 "intersects takes segment queries (intersects_mesh, kernels.hpp:80)");
            need(mesh->g.n_obj == 1, "the argument must be a mesh (one object)");
            tdb::run_queries_direct(ctx(), op, q, n, kind == TDB_QUERY_POINTS ? tdb::kQueryPoints : tdb::kQuerySegments,
                                    mesh->g, dist, hit, face);
        });
    tdb_queries qs = nullptr;
    int rc = tdb_queries_upload(q, n, kind, &qs);
    if (rc == TDB_OK)
        rc = op == TDB_OP_DISTANCE ? tdb_queries_mesh_distance(qs, mesh, dist, face)
                                   : tdb_queries_mesh_intersects(qs, mesh, hit, face);
    const std::string err = t_err;
    tdb_queries_free(qs);
    t_err = err;
    return rc;
}

int tdb_literal_table_eval(int op, int literal_kind, const double* literal, tdb_table records, double* dist_out,
                           uint8_t* hit_out, uint64_t* face_out) {
    return guarded([&] {
        need(records != nullptr && literal != nullptr, "null argument");
        need(op == TDB_OP_DISTANCE || op == TDB_OP_INTERSECTS, "unknown op");
        need(literal_kind == TDB_QUERY_SEGMENTS || literal_kind == TDB_QUERY_POINTS, "unknown literal kind");
        tdb::Ctx c = ctx();
        tdb::QuerySet q1;
        q1.device = t_device;
        try {
            tdb::queries_build(&q1, literal, 1, literal_kind == TDB_QUERY_SEGMENTS ? tdb::kQuerySegments
                                                                                    : tdb::kQueryPoints,
                               c.stream);
            tdb::run_literal_table(c, op, q1, records->g, dist_out, hit_out, face_out);
        } catch (...) {
            cudaFreeAsync(q1.planes, c.stream);
            throw;
        }
        cudaFreeAsync(q1.planes, c.stream);
    });
}

int tdb_segments_mesh_distance(const double* seg6, uint64_t n, tdb_mesh mesh, double* dist_out, uint64_t* face_out) {
    return one_shot_queries(seg6, n, TDB_QUERY_SEGMENTS, TDB_OP_DISTANCE, mesh, dist_out, nullptr, face_out);
}

int tdb_points_mesh_distance(const double* pt3, uint64_t n, tdb_mesh mesh, double* dist_out, uint64_t* face_out) {
    return one_shot_queries(pt3, n, TDB_QUERY_POINTS, TDB_OP_DISTANCE, mesh, dist_out, nullptr, face_out);
}

int tdb_segments_mesh_intersects(const double* seg6, uint64_t n, tdb_mesh mesh, uint8_t* hit_out, uint64_t* face_out) {
    return one_shot_queries(seg6, n, TDB_QUERY_SEGMENTS, TDB_OP_INTERSECTS, mesh, nullptr, hit_out, face_out);
}

int tdb_mesh_volume(tdb_mesh m, uint64_t chunk_size, double* volume_out) {
    return guarded([&] {
        need(m && volume_out, "null argument");
        need(m->g.n_obj == 1, "volume takes a mesh (one object)");
        *volume_out = tdb::run_volume(ctx(), m->g, chunk_size);
    });
}

int tdb_table_volume(tdb_table t, uint64_t chunk_size, double* volume_out) {
    return guarded([&] {
        need(t != nullptr && (volume_out != nullptr || t->g.n_obj == 0), "null argument");
        tdb::run_volume_table(ctx(), t->g, chunk_size, volume_out);
    });
}

int tdb_fp64_peak(double* tflops, double* ms) {
    return guarded([&] {
        need(tflops != nullptr, "null output");
        *tflops = tdb::fp64_peak(ctx(), ms);
    });
}

}  // extern "C"

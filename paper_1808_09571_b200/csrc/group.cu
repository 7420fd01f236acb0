// Device group: one process driving several B200s (SURVEY.md 8(b)
// "tdb_init(int n_gpus): NCCL comm + streams", 8(e)).
//
// The reference engine is a single process that calls run_batch from one
// thread per connection (pg_server.cpp:231,496); to spread one operator over
// the GPUs of a box the library itself owns the devices:
//   * one worker thread per device, bound to it with tdb_init (every per-
//     device call then runs the single-GPU path on that thread's stream);
//   * geometry is replicated: each member holds the whole store (B is needed
//     everywhere, and A's rows are addressed by global index so pair indices
//     stay i*|B|+j on every device);
//   * mesh x mesh splits A's rows into contiguous, tile-aligned ranges
//     (shard.py row_shards); a table splits its objects into contiguous
//     ranges of near-equal face count (shard.py object_shards);
//   * the only exchange is an NCCL MIN all-reduce over the members'
//     communicators (ncclCommInitAll: NVLink/NVSwitch on a B200 box):
//     distance = MIN of the distance bits (non-negative doubles order as
//     int64), then MIN of the pair among the members holding that distance
//     (the lexicographic (distance, pair) minimum: lowest pair on ties,
//     kernels.cpp:359,368-376); intersects = MIN of the lowest hit pair
//     (kernels.cpp:407-432). Table slices need no exchange: each member
//     writes its own rows of the caller's arrays.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "runtime.h"

namespace {

constexpr int64_t kNone = INT64_MAX;  // "no pair" inside the int64 reductions

#define NCK(expr)                                                                                  \
    do {                                                                                           \
        ncclResult_t r_ = (expr);                                                                  \
        if (r_ != ncclSuccess)                                                                     \
            throw ::tdb::CudaError(std::string(#expr) + ": " + ncclGetErrorString(r_));            \
    } while (0)

// One thread per device; run() hands every worker its member index and waits.
class Workers {
  public:
    explicit Workers(const std::vector<int>& devices) : n_((int)devices.size()), rc_(n_), msg_(n_) {
        for (int r = 0; r < n_; ++r) th_.emplace_back([this, r, dev = devices[r]] { loop(r, dev); });
        run([](int) { return TDB_OK; });  // wait until every worker bound its device
    }
    ~Workers() {
        {
            std::lock_guard<std::mutex> g(m_);
            stop_ = true;
            ++gen_;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    // f(member) returns a TDB status; the first failure (by member) is
    // reported with its message.
    int run(const std::function<int(int)>& f) {
        std::unique_lock<std::mutex> g(m_);
        job_ = &f;
        left_ = n_;
        ++gen_;
        cv_.notify_all();
        done_.wait(g, [this] { return left_ == 0; });
        job_ = nullptr;
        for (int r = 0; r < n_; ++r)
            if (rc_[r] != TDB_OK) return tdb::set_error(rc_[r], "device group member " + std::to_string(r) + ": " + msg_[r]);
        return TDB_OK;
    }

  private:
    void loop(int r, int dev) {
        int brc = tdb_init(dev);
        cudaStream_t own = nullptr;  // the member's launch stream
        if (brc == TDB_OK && cudaStreamCreateWithFlags(&own, cudaStreamNonBlocking) != cudaSuccess)
            brc = tdb::set_error(TDB_E_CUDA, cudaGetErrorString(cudaGetLastError()));
        if (brc == TDB_OK) brc = tdb_set_stream(own);
        const std::string bmsg = brc == TDB_OK ? "" : tdb_last_error();
        uint64_t seen = 0;
        for (;;) {
            const std::function<int(int)>* f;
            {
                std::unique_lock<std::mutex> g(m_);
                cv_.wait(g, [&] { return gen_ != seen; });
                seen = gen_;
                if (stop_) {
                    if (own) cudaStreamDestroy(own);
                    return;
                }
                f = job_;
            }
            int rc = brc;
            std::string msg = bmsg;
            if (rc == TDB_OK) {
                rc = (*f)(r);
                if (rc != TDB_OK) msg = tdb_last_error();
            }
            std::lock_guard<std::mutex> g(m_);
            rc_[r] = rc;
            msg_[r] = msg;
            if (--left_ == 0) done_.notify_all();
        }
    }
    int n_;
    std::vector<std::thread> th_;
    std::vector<int> rc_;
    std::vector<std::string> msg_;
    std::mutex m_;
    std::condition_variable cv_, done_;
    const std::function<int(int)>* job_ = nullptr;
    int left_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

// shard.py row_shards: contiguous kTile-aligned [begin, end) ranges
std::pair<uint64_t, uint64_t> row_shard(uint64_t n_rows, int world, int r) {
    const uint64_t tiles = (n_rows + tdb::kTile - 1) / tdb::kTile;
    const uint64_t t0 = tiles * (uint64_t)r / (uint64_t)world, t1 = tiles * (uint64_t)(r + 1) / (uint64_t)world;
    return {std::min(n_rows, t0 * tdb::kTile), std::min(n_rows, t1 * tdb::kTile)};
}

// shard.py object_shards: contiguous object ranges of near-equal face count
std::pair<uint64_t, uint64_t> object_shard(const std::vector<uint64_t>& off, int world, int r) {
    const uint64_t n_obj = off.size() - 1, total = off.back();
    auto cut = [&](int k) -> uint64_t {
        if (k <= 0) return 0;
        if (k >= world) return n_obj;
        const uint64_t target = total * (uint64_t)k / (uint64_t)world;
        // first object whose start is >= target (searchsorted left on off[:-1])
        return (uint64_t)(std::lower_bound(off.begin(), off.end() - 1, target) - off.begin());
    };
    uint64_t lo = cut(r), hi = cut(r + 1);
    return {std::min(lo, n_obj), std::min(std::max(hi, lo), n_obj)};
}

}  // namespace

struct tdb_group_s {
    std::vector<int> devices;
    // TDB_GROUP_SHARED_DEVICES=1 (tests only): members may share a device;
    // NCCL refuses duplicate devices in a communicator, so the MIN reductions
    // then run through host memory. The NCCL path is the product path.
    bool host_reduce = false;
    std::mutex red_mu;
    std::condition_variable red_cv;
    int red_cnt = 0;
    uint64_t red_gen = 0;
    int64_t red_acc = 0, red_val = 0;
    std::vector<ncclComm_t> comms;
    std::vector<int64_t*> scratch;  // one int64 per member for the all-reduces
    std::vector<tdb_stats> stats;   // per member, of the last group call
    // intersects early exit across devices: one lowest-hit word on member 0's
    // device, reached by the others through peer access (NVLink); off when a
    // member cannot map it
    unsigned long long* shared_hit = nullptr;
    bool early_exit = false;
    Workers* workers = nullptr;
    std::mutex call_mu;             // one group call at a time (NCCL ordering)
};

struct tdb_gmesh_s {
    tdb_group group;
    std::vector<tdb_geom_s*> member;  // one replica per device
    uint64_t n = 0, n_obj = 0;
    std::vector<uint64_t> off;
};

namespace {

// MIN all-reduce of one int64 across the group (member r's contribution v).
int64_t allreduce_min(tdb_group g, int r, int64_t v) {
    if (g->host_reduce) {
        std::unique_lock<std::mutex> lk(g->red_mu);
        const uint64_t gen = g->red_gen;
        g->red_acc = g->red_cnt == 0 ? v : std::min(g->red_acc, v);
        if (++g->red_cnt == (int)g->devices.size()) {
            g->red_val = g->red_acc;
            g->red_cnt = 0;
            ++g->red_gen;
            g->red_cv.notify_all();
        } else {
            g->red_cv.wait(lk, [&] { return g->red_gen != gen; });
        }
        return g->red_val;
    }
    cudaStream_t st = tdb::call_stream();
    CK(cudaMemcpyAsync(g->scratch[r], &v, sizeof v, cudaMemcpyHostToDevice, st));
    NCK(ncclAllReduce(g->scratch[r], g->scratch[r], 1, ncclInt64, ncclMin, g->comms[r], st));
    int64_t out = 0;
    CK(cudaMemcpyAsync(&out, g->scratch[r], sizeof out, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return out;
}

template <class F>
int member_guard(F&& f) {
    try {
        return f();
    } catch (const std::exception& e) {
        return tdb::set_error(TDB_E_CUDA, e.what());
    }
}

int upload_all(tdb_group g, const double* tri9, uint64_t n, const uint64_t* off, uint64_t n_obj, tdb_gmesh* out) {
    if (!g || !out) return tdb::set_error(TDB_E_ARG, "null argument");
    std::lock_guard<std::mutex> lk(g->call_mu);
    auto* m = new tdb_gmesh_s();
    m->group = g;
    m->member.assign(g->devices.size(), nullptr);
    m->n = n;
    m->n_obj = n_obj;
    m->off.assign(off, off + n_obj + 1);
    const int rc = g->workers->run([&](int r) {
        return off == nullptr || n_obj == 1 ? tdb_mesh_upload(tri9, n, &m->member[r])
                                            : tdb_table_upload(tri9, off, n_obj, &m->member[r]);
    });
    if (rc != TDB_OK) {
        const std::string err = tdb_last_error();
        tdb_gmesh_free(m);
        return tdb::set_error(rc, err);
    }
    *out = m;
    return TDB_OK;
}

}  // namespace

extern "C" {

int tdb_group_create(int n_devices, const int* devices, tdb_group* out) {
    if (!out || n_devices <= 0) return tdb::set_error(TDB_E_ARG, "need n_devices >= 1 and an output handle");
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count <= 0) {
        cudaGetLastError();
        return tdb::set_error(TDB_E_CUDA, "no CUDA device");
    }
    auto* g = new tdb_group_s();
    for (int r = 0; r < n_devices; ++r) {
        const int d = devices ? devices[r] : r;
        if (d < 0 || d >= count) {
            delete g;
            return tdb::set_error(TDB_E_ARG, "device index out of range");
        }
        for (int q : g->devices)
            if (q == d) g->host_reduce = true;
        g->devices.push_back(d);
    }
    if (g->host_reduce) {
        const char* e = getenv("TDB_GROUP_SHARED_DEVICES");
        if (!e || std::strcmp(e, "1") != 0) {
            delete g;
            return tdb::set_error(TDB_E_ARG, "a device may appear once in a group");
        }
    }
    g->comms.assign(n_devices, nullptr);
    g->scratch.assign(n_devices, nullptr);
    g->stats.assign(n_devices, tdb_stats{});
    const ncclResult_t nr = g->host_reduce ? ncclSuccess : ncclCommInitAll(g->comms.data(), n_devices, g->devices.data());
    if (nr != ncclSuccess) {
        const std::string msg = std::string("ncclCommInitAll: ") + ncclGetErrorString(nr);
        delete g;
        return tdb::set_error(TDB_E_CUDA, msg);
    }
    g->workers = new Workers(g->devices);
    std::vector<int> peer_ok(n_devices, 0);
    const int rc = g->workers->run([&](int r) {
        return member_guard([&] {
            CK(cudaMalloc(&g->scratch[r], sizeof(int64_t)));
            if (r == 0) {
                CK(cudaMalloc(&g->shared_hit, sizeof(unsigned long long)));
                peer_ok[r] = 1;
            } else if (g->devices[r] == g->devices[0]) {
                peer_ok[r] = 1;
            } else {
                int can = 0;
                CK(cudaDeviceCanAccessPeer(&can, g->devices[r], g->devices[0]));
                if (can) {
                    const cudaError_t e = cudaDeviceEnablePeerAccess(g->devices[0], 0);
                    if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
                    else CK(e);
                }
                peer_ok[r] = can;
            }
            return TDB_OK;
        });
    });
    g->early_exit = std::all_of(peer_ok.begin(), peer_ok.end(), [](int x) { return x != 0; });
    if (rc != TDB_OK) {
        const std::string err = tdb_last_error();
        tdb_group_free(g);
        return tdb::set_error(rc, err);
    }
    *out = g;
    return TDB_OK;
}

void tdb_group_free(tdb_group g) {
    if (!g) return;
    if (g->workers)
        g->workers->run([&](int r) {
            if (g->scratch[r]) cudaFree(g->scratch[r]);
            if (r == 0 && g->shared_hit) cudaFree(g->shared_hit);
            return TDB_OK;
        });
    delete g->workers;
    for (ncclComm_t c : g->comms)
        if (c) ncclCommDestroy(c);
    delete g;
}

int tdb_group_size(tdb_group g) { return g ? (int)g->devices.size() : 0; }

int tdb_group_mesh_upload(tdb_group g, const double* tri9, uint64_t n_tris, tdb_gmesh* out) {
    const uint64_t off[2] = {0, n_tris};
    return upload_all(g, tri9, n_tris, off, 1, out);
}

int tdb_group_table_upload(tdb_group g, const double* tri9, const uint64_t* face_offsets, uint64_t n_objects,
                           tdb_gmesh* out) {
    if (!face_offsets) return tdb::set_error(TDB_E_ARG, "null face offsets");
    return upload_all(g, tri9, face_offsets[n_objects], face_offsets, n_objects, out);
}

void tdb_gmesh_free(tdb_gmesh m) {
    if (!m) return;
    for (tdb_geom_s* h : m->member) tdb_mesh_free(h);  // frees on the handle's own device
    delete m;
}

int tdb_group_mesh_mesh_distance(tdb_group g, tdb_gmesh a, tdb_gmesh b, tdb_dist_out* out) {
    if (!g || !a || !b || !out) return tdb::set_error(TDB_E_ARG, "null argument");
    if (a->group != g || b->group != g) return tdb::set_error(TDB_E_ARG, "geometry belongs to another group");
    if (b->n_obj != 1) return tdb::set_error(TDB_E_ARG, "second argument must be a mesh (one object)");
    std::lock_guard<std::mutex> lk(g->call_mu);
    const int world = (int)g->devices.size();
    std::vector<tdb_dist_out> part(world);
    std::vector<int64_t> gd(world), gp(world);
    const int rc = g->workers->run([&](int r) {
        const auto [r0, r1] = row_shard(a->n, world, r);
        const int crc = tdb_mesh_mesh_distance_rows(a->member[r], r0, r1, b->member[r], &part[r]);
        tdb_last_stats(&g->stats[r]);
        return member_guard([&] {
            // every member joins both collectives, failed or not
            int64_t d = kNone;
            if (crc == TDB_OK && part[r].found) std::memcpy(&d, &part[r].distance, sizeof d);
            gd[r] = allreduce_min(g, r, d);
            gp[r] = allreduce_min(g, r, d == gd[r] && d != kNone ? (int64_t)part[r].pair : kNone);
            return crc == TDB_OK ? TDB_OK : tdb::set_error(crc, tdb_last_error());
        });
    });
    if (rc != TDB_OK) return rc;
    std::memset(out, 0, sizeof *out);
    out->distance = tdb::pos_inf_h();
    out->pair = out->i = out->j = UINT64_MAX;
    if (gd[0] == kNone) return TDB_OK;
    for (int r = 0; r < world; ++r)
        if (part[r].found && (int64_t)part[r].pair == gp[0]) {  // the owner's witnesses
            *out = part[r];
            break;
        }
    return TDB_OK;
}

int tdb_group_mesh_mesh_intersects(tdb_group g, tdb_gmesh a, tdb_gmesh b, tdb_hit_out* out) {
    if (!g || !a || !b || !out) return tdb::set_error(TDB_E_ARG, "null argument");
    if (a->group != g || b->group != g) return tdb::set_error(TDB_E_ARG, "geometry belongs to another group");
    if (b->n_obj != 1) return tdb::set_error(TDB_E_ARG, "second argument must be a mesh (one object)");
    std::lock_guard<std::mutex> lk(g->call_mu);
    const int world = (int)g->devices.size();
    std::vector<tdb_hit_out> part(world);
    std::vector<int64_t> gp(world);
    if (g->early_exit) {  // reset the shared lowest-hit word before any member starts
        const int irc = g->workers->run([&](int r) {
            return member_guard([&] {
                if (r == 0) {
                    CK(cudaMemsetAsync(g->shared_hit, 0xff, sizeof(unsigned long long), tdb::call_stream()));
                    CK(cudaStreamSynchronize(tdb::call_stream()));
                }
                return TDB_OK;
            });
        });
        if (irc != TDB_OK) return irc;
    }
    const int rc = g->workers->run([&](int r) {
        const auto [r0, r1] = row_shard(a->n, world, r);
        tdb::set_shared_hit(g->early_exit ? g->shared_hit : nullptr);
        const int crc = tdb_mesh_mesh_intersects_rows(a->member[r], r0, r1, b->member[r], &part[r]);
        tdb::set_shared_hit(nullptr);
        tdb_last_stats(&g->stats[r]);
        return member_guard([&] {
            gp[r] = allreduce_min(g, r, crc == TDB_OK && part[r].hit ? (int64_t)part[r].pair : kNone);
            return crc == TDB_OK ? TDB_OK : tdb::set_error(crc, tdb_last_error());
        });
    });
    if (rc != TDB_OK) return rc;
    std::memset(out, 0, sizeof *out);
    out->pair = out->i = out->j = UINT64_MAX;
    if (gp[0] == kNone) return TDB_OK;
    out->hit = 1;
    out->pair = (uint64_t)gp[0];
    const uint64_t nb = b->n;
    out->i = out->pair / nb;
    out->j = out->pair % nb;
    return TDB_OK;
}

int tdb_group_table_eval(tdb_group g, int op, tdb_gmesh records, tdb_gmesh literal, double* dist_out,
                         uint8_t* hit_out, uint64_t* pair_out) {
    if (!g || !records || !literal) return tdb::set_error(TDB_E_ARG, "null argument");
    if (records->group != g || literal->group != g) return tdb::set_error(TDB_E_ARG, "geometry belongs to another group");
    std::lock_guard<std::mutex> lk(g->call_mu);
    const int world = (int)g->devices.size();
    return g->workers->run([&](int r) {
        const auto [o0, o1] = object_shard(records->off, world, r);
        if (o0 == o1) {
            g->stats[r] = tdb_stats{};
            return TDB_OK;
        }
        const int rc = tdb_table_eval_rows(op, records->member[r], o0, o1, literal->member[r],
                                           dist_out ? dist_out + o0 : nullptr, hit_out ? hit_out + o0 : nullptr,
                                           pair_out ? pair_out + o0 : nullptr);
        tdb_last_stats(&g->stats[r]);
        return rc;
    });
}

int tdb_group_last_stats(tdb_group g, int member, tdb_stats* out) {
    if (!g || !out || member < 0 || member >= (int)g->devices.size())
        return tdb::set_error(TDB_E_ARG, "bad group member");
    *out = g->stats[member];
    return TDB_OK;
}

}  // extern "C"

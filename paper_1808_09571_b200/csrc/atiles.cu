// A side of the shared candidates: the distinct edges and
// vertices of each "super-tile" — kSuperTile consecutive 128-face tiles of
// one object — each listed with (at most) two of the tiles whose faces have
// it (a vertex in more tiles gets one entry per two tiles).
//
// Deduplicating within a super-tile instead of within a tile shares the
// edges between tiles too: a 1024-wide terrain's 128-face tiles are strips
// of one grid row, 2.0 distinct edges per face each, while a super-tile of
// 256 tiles (16 rows) has 1.53. The edge kernel attributes an entry's
// candidate to both of its tiles' items.
//
// Build (once per store, on the device): corner keys (super-tile, x, y, z
// bits) are radix-sorted (four stable passes), equal runs give vertex ids;
// edge keys (min id, max id) are sorted, and each run of faces sharing an
// edge becomes ceil(len / 2) entries (two tiles each; a manifold edge has one
// run of two). Ids are ordered by super-tile, so the entries of a super-tile
// are contiguous: per-super-tile offsets select a call's tiles.
#include <algorithm>
#include <cmath>
#include <vector>

#include <cub/cub.cuh>

#include "runtime.h"

namespace tdb {

namespace {

constexpr unsigned kNoSt = 0xffffffffu;

__global__ void face_tile_kernel(const Tile* __restrict__ tiles, uint64_t n_tiles, uint32_t* __restrict__ face_tile) {
    const uint64_t t = blockIdx.x;
    if (t >= n_tiles) return;
    const Tile T = tiles[t];
    for (uint32_t i = threadIdx.x; i < T.count; i += blockDim.x) face_tile[T.row0 + i] = (uint32_t)t;
}

// corners c = 3f + k: coordinate keys, super-tile key (kNoSt for degenerate
// faces: sorted last, no edges)
__global__ void corner_kernel(const double* __restrict__ planes, uint64_t n, uint64_t n_pad,
                              const uint32_t* __restrict__ face_tile, const uint32_t* __restrict__ tile_st,
                              unsigned long long* __restrict__ kx, unsigned long long* __restrict__ ky,
                              unsigned long long* __restrict__ kz, uint32_t* __restrict__ kst,
                              uint32_t* __restrict__ idx) {
    const uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= 3 * n) return;
    const uint64_t f = c / 3, k = c - 3 * f;
    const bool live = planes[(uint64_t)F_DEG * n_pad + f] == 0.0;
    kx[c] = (unsigned long long)__double_as_longlong(planes[(uint64_t)(F_V + 3 * k) * n_pad + f]);
    ky[c] = (unsigned long long)__double_as_longlong(planes[(uint64_t)(F_V + 3 * k + 1) * n_pad + f]);
    kz[c] = (unsigned long long)__double_as_longlong(planes[(uint64_t)(F_V + 3 * k + 2) * n_pad + f]);
    kst[c] = live ? tile_st[face_tile[f]] : kNoSt;
    idx[c] = (uint32_t)c;
}

template <class K>
__global__ void gather_kernel(const K* __restrict__ src, const uint32_t* __restrict__ idx, uint64_t m,
                              K* __restrict__ dst) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) dst[i] = src[idx[i]];
}

// sorted corner i starts a new vertex when its (st, x, y, z) differs from i-1
__global__ void vflag_kernel(const uint32_t* __restrict__ idx, uint64_t m, const unsigned long long* __restrict__ kx,
                             const unsigned long long* __restrict__ ky, const unsigned long long* __restrict__ kz,
                             const uint32_t* __restrict__ kst, uint32_t* __restrict__ flag) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const uint32_t a = idx[i];
    if (i == 0) {
        flag[i] = 1;
        return;
    }
    const uint32_t b = idx[i - 1];
    flag[i] = kst[a] != kst[b] || kx[a] != kx[b] || ky[a] != ky[b] || kz[a] != kz[b];
}

__global__ void vid_scatter_kernel(const uint32_t* __restrict__ idx, const uint32_t* __restrict__ vid_sorted,
                                   uint64_t m, uint32_t* __restrict__ vid) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) vid[idx[i]] = vid_sorted[i] - 1;  // inclusive scan of flags: ids from 1
}

// edge (f, k): V_k -> V_k+1, keyed by the unordered vertex id pair
__global__ void ekey_kernel(const uint32_t* __restrict__ vid, const uint32_t* __restrict__ kst, uint64_t n,
                            unsigned long long* __restrict__ key, uint32_t* __restrict__ val) {
    const uint64_t c = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= 3 * n) return;
    const uint64_t f = c / 3, k = c - 3 * f;
    const uint32_t a = vid[c], b = vid[3 * f + (k == 2 ? 0 : k + 1)];
    key[c] = kst[c] == kNoSt ? ~0ull : (unsigned long long)min(a, b) << 32 | max(a, b);
    val[c] = (uint32_t)c;
}

// run starts (as their index, else 0; a max-scan gives each element its run
// start) and entry flags (even offset within the run)
__global__ void run_kernel(const unsigned long long* __restrict__ key, uint64_t m, uint32_t* __restrict__ start) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) start[i] = (i == 0 || key[i] != key[i - 1]) ? (uint32_t)i : 0u;
}

__global__ void eflag_kernel(const unsigned long long* __restrict__ key, const uint32_t* __restrict__ start,
                             uint64_t m, uint32_t* __restrict__ flag) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) flag[i] = key[i] != ~0ull && ((i - start[i]) & 1) == 0;
}

// entry at sorted position i (an even offset in its run): the run's first
// edge (its face's direction) for the geometry, tiles of elements i and i+1
__global__ void entry_kernel(const double* __restrict__ planes, uint64_t n_pad,
                             const unsigned long long* __restrict__ key, const uint32_t* __restrict__ val,
                             const uint32_t* __restrict__ start, const uint32_t* __restrict__ flag,
                             const uint32_t* __restrict__ pos, uint64_t m, const uint32_t* __restrict__ face_tile,
                             const uint32_t* __restrict__ tile_st, double* __restrict__ out,
                             unsigned long long* __restrict__ st_count) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m || !flag[i]) return;
    const uint32_t rc = val[start[i]];
    const uint64_t f = rc / 3, k = rc - 3 * f;
    const uint32_t ta = face_tile[val[i] / 3];
    const uint32_t tb = (i + 1 < m && key[i + 1] == key[i]) ? face_tile[val[i + 1] / 3] : ta;
    double* p = out + (uint64_t)pos[i] * kAER;
    p[AR_Q] = planes[(uint64_t)(F_V + 3 * k) * n_pad + f];
    p[AR_Q + 1] = planes[(uint64_t)(F_V + 3 * k + 1) * n_pad + f];
    p[AR_Q + 2] = planes[(uint64_t)(F_V + 3 * k + 2) * n_pad + f];
#pragma unroll
    for (int c = 0; c < 3; ++c) p[AR_E + c] = planes[(uint64_t)(F_E + 3 * k + c) * n_pad + f];
    p[AR_L] = planes[(uint64_t)(F_L + k) * n_pad + f];
    p[AR_IL] = planes[(uint64_t)(F_IL + k) * n_pad + f];
    p[AR_TILE] = __longlong_as_double((long long)((unsigned long long)tb << 32 | ta));
    p[AR_TILE + 1] = 0.0;
    atomicAdd(st_count + tile_st[ta], 1ull);
}

// vertex entries. Sorted corner i: its vertex run starts at vstart[i]
// (max-scan); a corner is "tile-new" when its tile differs from the previous
// corner's in the run (corners of a run are in face order, so tiles ascend).
// Tile-new corners at an even rank in their run become entries carrying
// their tile and the next tile-new corner's (one entry per two tiles).
__global__ void vstart_kernel(const uint32_t* __restrict__ vflag, uint64_t m, uint32_t* __restrict__ vs) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) vs[i] = vflag[i] ? (uint32_t)i : 0u;
}

__global__ void tnew_kernel(const uint32_t* __restrict__ cur, const uint32_t* __restrict__ vstart, uint64_t m,
                            const uint32_t* __restrict__ face_tile, const uint32_t* __restrict__ kst,
                            uint32_t* __restrict__ tnew) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const uint32_t c = cur[i];
    tnew[i] = kst[c] != kNoSt && (vstart[i] == i || face_tile[c / 3] != face_tile[cur[i - 1] / 3]);
}

__global__ void vflag2_kernel(const uint32_t* __restrict__ tnew, const uint32_t* __restrict__ rank,
                              const uint32_t* __restrict__ vstart, uint64_t m, uint32_t* __restrict__ vent) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) vent[i] = tnew[i] && ((rank[i] - rank[vstart[i]]) & 1) == 0;
}

__global__ void ventry_kernel(const double* __restrict__ planes, uint64_t n_pad, const uint32_t* __restrict__ cur,
                              const uint32_t* __restrict__ vstart, const uint32_t* __restrict__ tnew,
                              const uint32_t* __restrict__ vent, const uint32_t* __restrict__ pos, uint64_t m,
                              const uint32_t* __restrict__ face_tile, const uint32_t* __restrict__ tile_st,
                              double* __restrict__ out, unsigned long long* __restrict__ st_count) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m || !vent[i]) return;
    const uint32_t c = cur[i];
    const uint64_t f = c / 3, k = c - 3 * f;
    const uint32_t ta = face_tile[f];
    uint32_t tb = ta;
    for (uint64_t j = i + 1; j < m && vstart[j] == vstart[i]; ++j)  // the next tile-new corner of the run
        if (tnew[j]) {
            tb = face_tile[cur[j] / 3];
            break;
        }
    double* p = out + (uint64_t)pos[i] * kAVR;
    p[0] = planes[(uint64_t)(F_V + 3 * k) * n_pad + f];
    p[1] = planes[(uint64_t)(F_V + 3 * k + 1) * n_pad + f];
    p[2] = planes[(uint64_t)(F_V + 3 * k + 2) * n_pad + f];
    p[3] = __longlong_as_double((long long)((unsigned long long)tb << 32 | ta));
    atomicAdd(st_count + tile_st[ta], 1ull);
}

// A-side entries reordered by their first tile, so that any tile range is
// (almost) a contiguous range: keys, per-tile counts, per-super-tile span of
// (second tile - first tile).
__global__ void tkey_kernel(const double* __restrict__ rec, uint64_t n, int stride, int field,
                            const uint32_t* __restrict__ tile_st, uint32_t* __restrict__ key,
                            uint32_t* __restrict__ idx, unsigned long long* __restrict__ tcount,
                            unsigned* __restrict__ span) {
    const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    const unsigned long long t = (unsigned long long)__double_as_longlong(rec[e * stride + field]);
    const uint32_t ta = (uint32_t)t, tb = (uint32_t)(t >> 32);
    key[e] = ta;
    idx[e] = (uint32_t)e;
    atomicAdd(tcount + ta, 1ull);
    atomicMax(span + tile_st[ta], tb - ta);
}

__global__ void rgather_kernel(const double* __restrict__ in, const uint32_t* __restrict__ idx, uint64_t n,
                               int stride, double* __restrict__ out) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n * stride) return;
    const uint64_t e = i / stride, k = i - e * stride;
    out[i] = in[(uint64_t)idx[e] * stride + k];
}

template <class T>
struct DevBuf {
    T* p = nullptr;
    cudaStream_t st;
    DevBuf(uint64_t n, cudaStream_t s) : st(s) { CK(cudaMallocAsync(&p, std::max<uint64_t>(n, 1) * sizeof(T), s)); }
    ~DevBuf() { cudaFreeAsync(p, st); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
};

struct MaxOp {
    __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const { return a > b ? a : b; }
};

}  // namespace

namespace {

// The lists of one grouping: groups of `group_tiles` consecutive tiles of one
// object; distinct edges (and, when asked, vertices) per group, each entry
// carrying two of its tiles; entries ordered by group.
struct SuperLists {
    std::vector<uint32_t> tile_grp;
    std::vector<uint64_t> eoff, voff;  // per group: first entry
    double* edges = nullptr;
    double* verts = nullptr;
};

void build_super(const Geom& g, uint64_t group_tiles, bool with_vertices, cudaStream_t st, SuperLists& L) {
    const uint64_t nt = g.h_tiles.size(), n = g.n, m = 3 * n;
    std::vector<uint32_t> tile_st(nt);
    uint32_t n_st = 0;
    for (uint64_t o = 0; o + 1 < g.obj_tile0.size(); ++o) {
        const uint64_t t0 = g.obj_tile0[o], t1 = g.obj_tile0[o + 1];
        for (uint64_t t = t0; t < t1; ++t) tile_st[t] = n_st + (uint32_t)((t - t0) / group_tiles);
        n_st += (uint32_t)((t1 - t0 + group_tiles - 1) / group_tiles);
    }
    L.tile_grp = tile_st;
    L.eoff.assign(n_st + 1, 0);
    L.voff.assign(n_st + 1, 0);
    if (nt == 0 || m == 0) return;
    if (m >= 0x7fffffffull)  // cub sorts / scans take int counts
        throw std::invalid_argument("shared-candidate lists: more than 2^31 face corners (715M faces) in one store");
    DevBuf<uint32_t> d_tile_st(nt, st), face_tile(n, st);
    CK(cudaMemcpyAsync(d_tile_st.p, tile_st.data(), nt * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    face_tile_kernel<<<(unsigned)nt, 128, 0, st>>>(g.d_tiles, nt, face_tile.p);
    CK(cudaGetLastError());
    DevBuf<unsigned long long> kx(m, st), ky(m, st), kz(m, st), ks(m, st);
    DevBuf<uint32_t> kst(m, st), idx(m, st), idx2(m, st), tmp32(m, st), vid(m, st);
    const unsigned grid = (unsigned)((m + 255) / 256);
    corner_kernel<<<grid, 256, 0, st>>>(g.planes, n, g.n_pad, face_tile.p, d_tile_st.p, kx.p, ky.p, kz.p, kst.p,
                                        idx.p);
    CK(cudaGetLastError());
    // LSD: z, y, x (64-bit), then the super-tile (32-bit); stable passes
    size_t tb = 0, tb2 = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, ks.p, ks.p, idx.p, idx2.p, (int)m, 0, 64, st));
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tb2, tmp32.p, tmp32.p, idx.p, idx2.p, (int)m, 0, 32, st));
    size_t tbs = 0;
    CK(cub::DeviceScan::InclusiveSum(nullptr, tbs, tmp32.p, tmp32.p, (int)m, st));
    size_t tbm = 0;
    CK(cub::DeviceScan::InclusiveScan(nullptr, tbm, tmp32.p, tmp32.p, MaxOp{}, (int)m, st));
    DevBuf<unsigned char> temp(std::max(std::max(tb, tb2), std::max(tbs, tbm)), st);
    const size_t tcap = std::max(std::max(tb, tb2), std::max(tbs, tbm));
    DevBuf<unsigned long long> ksorted(m, st);
    uint32_t* cur = idx.p;
    uint32_t* nxt = idx2.p;
    for (const unsigned long long* key : {kz.p, ky.p, kx.p}) {
        gather_kernel<<<grid, 256, 0, st>>>(key, cur, m, ks.p);
        CK(cudaGetLastError());
        size_t t = tcap;
        CK(cub::DeviceRadixSort::SortPairs(temp.p, t, ks.p, ksorted.p, cur, nxt, (int)m, 0, 64, st));
        std::swap(cur, nxt);
    }
    {
        gather_kernel<<<grid, 256, 0, st>>>(kst.p, cur, m, tmp32.p);
        CK(cudaGetLastError());
        DevBuf<uint32_t> stsorted(m, st);
        size_t t = tcap;
        CK(cub::DeviceRadixSort::SortPairs(temp.p, t, tmp32.p, stsorted.p, cur, nxt, (int)m, 0, 32, st));
        std::swap(cur, nxt);
    }
    // vertex ids (ordered by super-tile)
    vflag_kernel<<<grid, 256, 0, st>>>(cur, m, kx.p, ky.p, kz.p, kst.p, tmp32.p);
    CK(cudaGetLastError());
    {
        size_t t = tcap;
        CK(cub::DeviceScan::InclusiveSum(temp.p, t, tmp32.p, nxt, (int)m, st));
    }
    vid_scatter_kernel<<<grid, 256, 0, st>>>(cur, nxt, m, vid.p);
    CK(cudaGetLastError());
    if (with_vertices) {  // vertex entries (tmp32 still holds the vertex-start flags)
        DevBuf<uint32_t> vs0(m, st), vstart(m, st), tnew(m, st), rank(m, st), vent(m, st), vpos(m, st);
        vstart_kernel<<<grid, 256, 0, st>>>(tmp32.p, m, vs0.p);
        CK(cudaGetLastError());
        size_t t = tcap;
        CK(cub::DeviceScan::InclusiveScan(temp.p, t, vs0.p, vstart.p, MaxOp{}, (int)m, st));
        tnew_kernel<<<grid, 256, 0, st>>>(cur, vstart.p, m, face_tile.p, kst.p, tnew.p);
        CK(cudaGetLastError());
        t = tcap;
        CK(cub::DeviceScan::ExclusiveSum(temp.p, t, tnew.p, rank.p, (int)m, st));
        vflag2_kernel<<<grid, 256, 0, st>>>(tnew.p, rank.p, vstart.p, m, vent.p);
        CK(cudaGetLastError());
        t = tcap;
        CK(cub::DeviceScan::ExclusiveSum(temp.p, t, vent.p, vpos.p, (int)m, st));
        uint32_t lp = 0, lf = 0;
        CK(cudaMemcpyAsync(&lp, vpos.p + m - 1, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&lf, vent.p + m - 1, 4, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        const uint64_t nv = (uint64_t)lp + lf;
        double* vout = nullptr;
        CK(cudaMallocAsync(&vout, std::max<uint64_t>(nv, 1) * kAVR * sizeof(double), st));
        DevBuf<unsigned long long> vcount(n_st, st);
        CK(cudaMemsetAsync(vcount.p, 0, std::max<uint32_t>(n_st, 1) * sizeof(unsigned long long), st));
        ventry_kernel<<<grid, 256, 0, st>>>(g.planes, g.n_pad, cur, vstart.p, tnew.p, vent.p, vpos.p, m, face_tile.p,
                                            d_tile_st.p, vout, vcount.p);
        CK(cudaGetLastError());
        std::vector<unsigned long long> cnt(n_st);
        CK(cudaMemcpyAsync(cnt.data(), vcount.p, n_st * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        for (uint32_t q = 0; q < n_st; ++q) L.voff[q + 1] = L.voff[q] + cnt[q];
        L.verts = vout;
    }
    // edges
    DevBuf<unsigned long long> ekey(m, st);
    ekey_kernel<<<grid, 256, 0, st>>>(vid.p, kst.p, n, ks.p, idx.p);
    CK(cudaGetLastError());
    {
        size_t t = tcap;
        CK(cub::DeviceRadixSort::SortPairs(temp.p, t, ks.p, ekey.p, idx.p, idx2.p, (int)m, 0, 64, st));
    }
    const uint32_t* val = idx2.p;
    run_kernel<<<grid, 256, 0, st>>>(ekey.p, m, tmp32.p);
    CK(cudaGetLastError());
    DevBuf<uint32_t> start(m, st), flag(m, st), pos(m, st);
    {
        size_t t = tcap;
        CK(cub::DeviceScan::InclusiveScan(temp.p, t, tmp32.p, start.p, MaxOp{}, (int)m, st));
    }
    eflag_kernel<<<grid, 256, 0, st>>>(ekey.p, start.p, m, flag.p);
    CK(cudaGetLastError());
    {
        size_t t = tcap;
        CK(cub::DeviceScan::ExclusiveSum(temp.p, t, flag.p, pos.p, (int)m, st));
    }
    uint32_t last_pos = 0, last_flag = 0;
    CK(cudaMemcpyAsync(&last_pos, pos.p + m - 1, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&last_flag, flag.p + m - 1, 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const uint64_t n_entries = (uint64_t)last_pos + last_flag;
    double* out = nullptr;
    CK(cudaMallocAsync(&out, std::max<uint64_t>(n_entries, 1) * kAER * sizeof(double), st));
    DevBuf<unsigned long long> st_count(n_st, st);
    CK(cudaMemsetAsync(st_count.p, 0, std::max<uint32_t>(n_st, 1) * sizeof(unsigned long long), st));
    entry_kernel<<<grid, 256, 0, st>>>(g.planes, g.n_pad, ekey.p, val, start.p, flag.p, pos.p, m, face_tile.p,
                                       d_tile_st.p, out, st_count.p);
    CK(cudaGetLastError());
    std::vector<unsigned long long> cnt(n_st);
    CK(cudaMemcpyAsync(cnt.data(), st_count.p, n_st * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (uint32_t s = 0; s < n_st; ++s) L.eoff[s + 1] = L.eoff[s] + cnt[s];
    L.edges = out;
}

}  // namespace

// Reorders n records (stride doubles, tiles in `field`) by their first tile;
// returns per-tile offsets (n_tiles + 1) and per-super-tile spans.
static double* by_tile(double* rec, uint64_t n, int stride, int field, const std::vector<uint32_t>& tile_st,
                       uint32_t n_st, cudaStream_t st, std::vector<uint64_t>& toff, std::vector<uint32_t>& span) {
    const uint64_t nt = tile_st.size();
    toff.assign(nt + 1, 0);
    span.assign(n_st, 0);
    if (n == 0) return rec;
    DevBuf<uint32_t> d_tst(nt, st), key(n, st), key2(n, st), idx(n, st), idx2(n, st);
    DevBuf<unsigned long long> cnt(nt, st);
    DevBuf<unsigned> d_span(n_st, st);
    CK(cudaMemcpyAsync(d_tst.p, tile_st.data(), nt * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
    CK(cudaMemsetAsync(cnt.p, 0, nt * sizeof(unsigned long long), st));
    CK(cudaMemsetAsync(d_span.p, 0, std::max<uint32_t>(n_st, 1) * sizeof(unsigned), st));
    tkey_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(rec, n, stride, field, d_tst.p, key.p, idx.p, cnt.p,
                                                             d_span.p);
    CK(cudaGetLastError());
    size_t tb = 0;
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, key.p, key2.p, idx.p, idx2.p, (int)n, 0, 32, st));
    DevBuf<unsigned char> temp(tb, st);
    CK(cub::DeviceRadixSort::SortPairs(temp.p, tb, key.p, key2.p, idx.p, idx2.p, (int)n, 0, 32, st));
    double* out = nullptr;
    CK(cudaMallocAsync(&out, n * stride * sizeof(double), st));
    rgather_kernel<<<(unsigned)((n * stride + 255) / 256), 256, 0, st>>>(rec, idx2.p, n, stride, out);
    CK(cudaGetLastError());
    CK(cudaFreeAsync(rec, st));
    std::vector<unsigned long long> c(nt);
    std::vector<unsigned> sp(n_st);
    CK(cudaMemcpyAsync(c.data(), cnt.p, nt * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(sp.data(), d_span.p, n_st * sizeof(unsigned), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (uint64_t t = 0; t < nt; ++t) toff[t + 1] = toff[t] + c[t];
    span.assign(sp.begin(), sp.end());
    return out;
}

void geom_super_tiles(const Geom& g, cudaStream_t st) {
    SuperLists L;
    build_super(g, kSuperTile, true, st, L);
    const uint32_t n_st = (uint32_t)(L.eoff.size() - 1);
    g.aedges = by_tile(L.edges, L.eoff.back(), kAER, AR_TILE, L.tile_grp, n_st, st, g.h_tile_eoff, g.h_st_espan);
    g.averts = by_tile(L.verts, L.voff.back(), kAVR, 3, L.tile_grp, n_st, st, g.h_tile_voff, g.h_st_vspan);
    g.h_tile_st = std::move(L.tile_grp);
    g.h_st_tile0.assign(n_st + 1, (uint64_t)g.h_tile_st.size());
    for (uint64_t t = g.h_tile_st.size(); t-- > 0;) g.h_st_tile0[g.h_tile_st[t]] = t;
}

// FP64 entries (kAER) -> FP32 records (kBER) relative to o.
__global__ void bedge_f32_kernel(const double* __restrict__ e, uint64_t n, double ox, double oy, double oz,
                                 float4* __restrict__ out) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double* r = e + i * kAER;
    out[2 * i] = make_float4((float)(r[AR_Q] - ox), (float)(r[AR_Q + 1] - oy), (float)(r[AR_Q + 2] - oz),
                             (float)r[AR_E]);
    out[2 * i + 1] = make_float4((float)r[AR_E + 1], (float)r[AR_E + 2], (float)r[AR_L], (float)r[AR_IL]);
}

void geom_super_bedges(const Geom& g, cudaStream_t st) {
    SuperLists L;
    build_super(g, kBSuper / kTile, false, st, L);
    g.h_bseoff = std::move(L.eoff);
    const uint64_t n = g.h_bseoff.back();
    // origin: B's box centre (its non-degenerate faces); every start point is
    // within the half-diagonal of it
    const double* s = g.stats;
    const bool box = std::isfinite(s[0]) && std::isfinite(s[1]) && std::isfinite(s[2]) && std::isfinite(s[3]) &&
                     std::isfinite(s[4]) && std::isfinite(s[5]);
    double r2 = 0.0;
    for (int k = 0; k < 3; ++k) {
        g.bse_org[k] = box ? 0.5 * (s[k] + s[3 + k]) : 0.0;
        r2 += box ? (s[3 + k] - s[k]) * (s[3 + k] - s[k]) : 0.0;
    }
    g.bse_rB = 0.5 * std::sqrt(r2) * (1.0 + 1e-12);
    CK(cudaMallocAsync(&g.bedges, std::max<uint64_t>(n, 1) * 2 * sizeof(float4), st));
    if (n) {
        bedge_f32_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(L.edges, n, g.bse_org[0], g.bse_org[1],
                                                                       g.bse_org[2], g.bedges);
        CK(cudaGetLastError());
    }
    CK(cudaFreeAsync(L.edges, st));
    CK(cudaMallocAsync(&g.d_bseoff, g.h_bseoff.size() * sizeof(uint64_t), st));
    CK(cudaMemcpyAsync(g.d_bseoff, g.h_bseoff.data(), g.h_bseoff.size() * sizeof(uint64_t), cudaMemcpyHostToDevice,
                       st));
}

}  // namespace tdb

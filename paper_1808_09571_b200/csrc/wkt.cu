// Device geometry loader: WKT text (TIN Z / POLYHEDRALSURFACE Z) parsed in
// HBM straight into the device store (north star "drop-in
// for ... its mesh/geometry loader").
//
// Replaces tindb::parse_wkt (wkt.hpp:35, wkt.cpp:188-231) + the TriangleMesh
// it returns, for one literal (load_wkt_file, store.cpp:133-160) or many
// (the WKT column of load_csv_text, store.cpp:71-122). The result is
// bit-identical to the reference: the same language is accepted, numbers
// convert exactly as std::from_chars (wkt_number.cuh), polygon patches are
// fan-triangulated from their first vertex (wkt.cpp:134-138), and a rejected
// literal reports the reference's WktParseError message and byte position.
//
// Pipeline (one batch of literals, <= 2 GiB of text):
//   1. host: each literal's header ("TIN Z" / "POLYHEDRALSURFACE Z"), a few
//      bytes, is read on the host; the bodies go to HBM in one copy;
//   2. lex (count, scan, emit): one thread per 32-byte span classifies bytes;
//      a maximal run of number characters [0-9.eE+-] is split into numbers
//      by the thread owning its first byte, with the from_chars grammar;
//      tokens are ( ) , and NUM; numbers are converted on the spot (rare
//      hard cases go to a big-integer pass);
//   3. grammar: token depth by prefix sum; every token checks its neighbours
//      against the surface grammar (a regular language over tokens once the
//      depth is known); rings are located by a second prefix sum;
//   4. rings: size, TIN-ness and closure checks; faces per ring (P - 3);
//   5. emit: fan triangles written AoS and handed to the store's prep pass.
// Any violation marks the literal; the host then re-reads that literal only
// to word the error exactly as the reference does (wkt_explain below) — the
// device decides acceptance and produces every coordinate.
#include <cub/cub.cuh>

#include <cctype>
#include <charconv>
#include <cmath>
#include <string>
#include <string_view>
#include <system_error>
#include <vector>

#include "runtime.h"
#include "wkt_number.cuh"

namespace tdb {

namespace {

enum : uint8_t { T_NONE = 0, T_LP = 1, T_RP = 2, T_CM = 3, T_NUM = 4 };
constexpr int kSpan = 32;                              // bytes per lexer thread
constexpr uint64_t kBatchBytes = (1ull << 31) - 1024;  // 32-bit token / number indices

__device__ __forceinline__ bool ws_byte(unsigned char c) { return c == ' ' || (c >= 9 && c <= 13); }
__device__ __forceinline__ bool num_byte(unsigned char c) {
    return (c >= '0' && c <= '9') || c == '.' || c == '-' || c == '+' || c == 'e' || c == 'E';
}

struct LexArgs {
    const char* text;
    uint64_t n;
    const uint64_t* bb;  // literal body [bb, be), sorted
    const uint64_t* be;
    uint32_t n_lit;
    uint32_t* cnt_tok;  // pass 0: per-thread counts; pass 1: exclusive offsets
    uint32_t* cnt_num;
    uint8_t* tok;
    uint32_t* tok_num;  // numbers before the token (its own index for NUM)
    double* nums;
    uint32_t* slow;  // number index, byte offset, length of hard numbers
    uint64_t* slow_pos;
    uint32_t* slow_len;
    unsigned int* n_slow;
    uint32_t* lit_tok0;
    unsigned long long* err_byte;
    uint8_t* span_multi;  // pass 0 -> 1: the span has a run with several numbers
};

constexpr int kLexThreads = 256;
constexpr int kLexChunk = kLexThreads * kSpan;  // bytes per CTA
constexpr int kLexHalo = 512;                   // run look-ahead kept in SMEM
constexpr int kTextPad = 16;                    // bytes before text[0] in the device copy

// Shared view of a CTA's text window: bytes [c0 - kTextPad, c0 + kLexChunk +
// kLexHalo) in SMEM, the rest read from global memory.
struct Window {
    const char* sm;
    const char* text;
    uint64_t c0, end;
    __device__ __forceinline__ const char* at(uint64_t i) const {
        return i < end ? sm + kTextPad + (i - c0) : text + i;
    }
    __device__ __forceinline__ bool in(uint64_t i) const { return i <= end; }
};

// Emit (PASS 1) or count (PASS 0) the number(s) of run [p, r) whose first
// token / number indices are tok / num; returns the number count, or -1 on
// a lexical error (PASS 0 records it).
template <int PASS>
__device__ int lex_run(const LexArgs& a, const Window& w, uint64_t p, uint64_t r, uint32_t tok, uint32_t num) {
    const bool smem = w.in(r);
    int cnt = 0;
    while (p < r) {  // from_chars maximal munch, number after number
        const num::Scan s = smem ? num::parse_number<PASS == 1>(w.at(p), w.at(r))
                                 : num::parse_number<PASS == 1>(a.text + p, a.text + r);
        if (s.status == num::kNoMatch || s.status == num::kRange) {
            if (!PASS) atomicMin(a.err_byte, (unsigned long long)p);
            return -1;
        }
        if (PASS) {
            a.tok[tok + cnt] = T_NUM;
            a.tok_num[tok + cnt] = num + cnt;
            if (s.status == num::kOk) {
                a.nums[num + cnt] = s.value;
            } else {
                const unsigned int q = atomicAdd(a.n_slow, 1u);
                a.slow[q] = num + cnt;
                a.slow_pos[q] = p;
                a.slow_len[q] = s.len;
            }
        }
        ++cnt;
        p += s.len;
    }
    return cnt;
}

constexpr int kMaxRuns = kSpan / 2;  // runs are separated by at least one byte

// Byte-by-byte lexing of one span (the reference order of work); used for
// spans where a run holds several numbers ("1-2"), which pass 0 flags.
template <int PASS>
__device__ void lex_span_serial(const LexArgs& a, const Window& w, uint64_t i0, uint64_t i1, int64_t j,
                                uint32_t tok0, uint32_t num0, uint32_t* ntok_out, uint32_t* nnum_out) {
    uint64_t cur_bb = j >= 0 ? a.bb[j] : 0, cur_be = j >= 0 ? a.be[j] : 0;
    uint64_t next_bb = j + 1 < (int64_t)a.n_lit ? a.bb[j + 1] : ~0ull;
    uint32_t ntok = 0, nnum = 0;
    for (uint64_t i = i0; i < i1; ++i) {
        while (i >= next_bb) {
            ++j;
            cur_bb = next_bb;
            cur_be = a.be[j];
            next_bb = j + 1 < (int64_t)a.n_lit ? a.bb[j + 1] : ~0ull;
        }
        if (j < 0 || i >= cur_be) continue;
        if (PASS && i == cur_bb) a.lit_tok0[j] = tok0 + ntok;
        const unsigned char c = (unsigned char)*w.at(i);
        if (ws_byte(c)) continue;
        if (c == '(' || c == ')' || c == ',') {
            if (PASS) {
                a.tok[tok0 + ntok] = c == '(' ? T_LP : c == ')' ? T_RP : T_CM;
                a.tok_num[tok0 + ntok] = num0 + nnum;
            }
            ++ntok;
            continue;
        }
        if (!num_byte(c)) {
            if (!PASS) atomicMin(a.err_byte, (unsigned long long)i);
            continue;
        }
        if (i > cur_bb && num_byte((unsigned char)*w.at(i - 1))) continue;  // run owned upstream
        uint64_t r = i + 1;
        while (r < cur_be && num_byte((unsigned char)*w.at(r))) ++r;
        const int c2 = lex_run<PASS>(a, w, i, r, tok0 + ntok, num0 + nnum);
        if (c2 > 0) ntok += c2, nnum += c2;
    }
    *ntok_out = ntok;
    *nnum_out = nnum;
}

// One CTA stages its 8 KB of text (+ halo, + the byte before) in SMEM with
// 16-byte loads. Each thread owns a 32-byte span and works in two phases so
// the lanes of a warp stay converged:
//   A. classify the span's bytes: structural tokens (written in pass 1), and
//      the extent of each run of number characters starting in the span;
//   B. parse the runs in lockstep (run k of every lane together).
// Token indices in phase A assume one number per run; pass 0 flags the spans
// where a run holds several ("1-2"), and pass 1 lexes those byte by byte.
template <int PASS>
__global__ void __launch_bounds__(kLexThreads) lex_kernel(LexArgs a) {
    __shared__ alignas(16) char sm[kTextPad + kLexChunk + kLexHalo];
    const uint64_t c0 = (uint64_t)blockIdx.x * kLexChunk;
    {
        const uint4* src = reinterpret_cast<const uint4*>(a.text + c0 - kTextPad);
        uint4* dst = reinterpret_cast<uint4*>(sm);
        for (int k = threadIdx.x; k < (kTextPad + kLexChunk + kLexHalo) / 16; k += kLexThreads) dst[k] = src[k];
    }
    __syncthreads();
    const Window w{sm, a.text, c0, c0 + kLexChunk + kLexHalo};
    const uint64_t t = (uint64_t)blockIdx.x * kLexThreads + threadIdx.x;
    const uint64_t i0 = t * kSpan;
    if (i0 >= a.n) return;
    const uint64_t i1 = min(a.n, i0 + kSpan);
    int64_t lo = 0, hi = a.n_lit;
    while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (a.bb[mid] <= i0) lo = mid + 1;
        else hi = mid;
    }
    const int64_t j0 = lo - 1;
    const uint32_t tok0 = PASS ? a.cnt_tok[t] : 0, num0 = PASS ? a.cnt_num[t] : 0;
    if (PASS && a.span_multi[t]) {
        uint32_t nt, nn;
        lex_span_serial<PASS>(a, w, i0, i1, j0, tok0, num0, &nt, &nn);
        return;
    }

    // ---- phase A
    uint8_t rs[kMaxRuns];   // run start, offset from i0
    uint8_t rb[kMaxRuns];   // structural tokens before the run
    uint16_t re[kMaxRuns];  // run end, offset from i0; 0xffff: still open at i1
    uint64_t open_be = 0;   // body end bounding the open run
    int nr = 0;
    uint32_t nstruct = 0;
    bool open = false;
    {
        int64_t j = j0;
        uint64_t cur_bb = j >= 0 ? a.bb[j] : 0, cur_be = j >= 0 ? a.be[j] : 0;
        uint64_t next_bb = j + 1 < (int64_t)a.n_lit ? a.bb[j + 1] : ~0ull;
        for (uint64_t i = i0; i < i1; ++i) {
            while (i >= next_bb) {
                if (open) re[nr - 1] = (uint16_t)(i - i0), open = false;
                ++j;
                cur_bb = next_bb;
                cur_be = a.be[j];
                next_bb = j + 1 < (int64_t)a.n_lit ? a.bb[j + 1] : ~0ull;
            }
            if (j < 0 || i >= cur_be) {
                if (open) re[nr - 1] = (uint16_t)(i - i0), open = false;
                continue;
            }
            if (PASS && i == cur_bb) a.lit_tok0[j] = tok0 + nstruct + nr;
            const unsigned char c = (unsigned char)sm[kTextPad + (i - c0)];
            const bool nb = num_byte(c);
            if (open) {
                if (nb) continue;
                re[nr - 1] = (uint16_t)(i - i0);
                open = false;
            }
            if (ws_byte(c)) continue;
            if (c == '(' || c == ')' || c == ',') {
                if (PASS) {
                    const uint32_t k = tok0 + nstruct + nr;
                    a.tok[k] = c == '(' ? T_LP : c == ')' ? T_RP : T_CM;
                    a.tok_num[k] = num0 + nr;
                }
                ++nstruct;
                continue;
            }
            if (!nb) {
                if (!PASS) atomicMin(a.err_byte, (unsigned long long)i);
                continue;
            }
            if (i > cur_bb && num_byte((unsigned char)sm[kTextPad + (i - c0) - 1])) continue;  // owned upstream
            rs[nr] = (uint8_t)(i - i0);
            rb[nr] = (uint8_t)nstruct;
            re[nr] = 0xffff;
            ++nr;
            open = true;
            open_be = cur_be;
        }
    }

    // ---- phase B
    uint32_t nnum = 0;
    bool multi = false;
    for (int k = 0; k < nr; ++k) {
        const uint64_t p = i0 + rs[k];
        uint64_t r;
        if (re[k] != 0xffff) {
            r = i0 + re[k];
        } else {
            r = i1;
            while (r < open_be && num_byte((unsigned char)*w.at(r))) ++r;
        }
        const int c = lex_run<PASS>(a, w, p, r, tok0 + rb[k] + nnum, num0 + nnum);
        if (c < 0) continue;
        multi |= c != 1;
        nnum += (uint32_t)c;
    }
    if (!PASS) {
        a.cnt_tok[t] = nstruct + nnum;
        a.cnt_num[t] = nnum;
        a.span_multi[t] = multi;
    }
}

__global__ void slow_number_kernel(const char* text, const uint32_t* slow, const uint64_t* pos, const uint32_t* len,
                                   const unsigned int* n_slow, double* nums, unsigned long long* err_byte) {
    const unsigned int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= *n_slow) return;
    const num::Scan s = num::parse_number_slow(text + pos[q], len[q]);
    if (s.status != num::kOk) atomicMin(err_byte, (unsigned long long)pos[q]);
    else nums[slow[q]] = s.value;
}

struct DepthDelta {
    __host__ __device__ __forceinline__ int operator()(uint8_t t) const {
        return t == T_LP ? 1 : t == T_RP ? -1 : 0;
    }
};

__device__ __forceinline__ uint32_t literal_of(const uint32_t* lit_tok0, uint32_t n_lit, uint32_t k) {
    uint32_t lo = 0, hi = n_lit;  // last literal whose first token <= k
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (lit_tok0[mid] <= k) lo = mid + 1;
        else hi = mid;
    }
    return lo ? lo - 1 : 0;
}

struct GramArgs {
    const uint8_t* tok;
    const int* depth;  // exclusive prefix of DepthDelta
    uint32_t T;
    const uint32_t* lit_tok0;  // n_lit + 1 entries
    uint32_t n_lit;
    uint32_t* ring_open;  // per token (+1): 1 at a ring's '('
    unsigned int* err_lit;
};

// Surface grammar, checked per token once depth d (before the token) is
// known — the reference's recursive descent (wkt.cpp:101-170) as local rules:
//   d=0 '(' first token; d=1 '(' after the opener or a d=1 ','; d=2 '(' after
//   a d=1 '(' and before a number; d=3 ')' after a number, before ')';
//   d=2 ')' after ')', before ',' or ')'; d=1 ')' after ')', last token;
//   d=3 ',' between numbers; d=1 ',' between ')' and '('; a number at d=3
//   that starts a point follows '(' or ',' and is followed by two numbers
//   and then ',' or ')'.
__global__ void grammar_kernel(GramArgs a) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= a.T) return;
    const uint32_t L = literal_of(a.lit_tok0, a.n_lit, k);
    const uint32_t first = a.lit_tok0[L], last = a.lit_tok0[L + 1] - 1;
    const uint8_t c = a.tok[k];
    const int d = a.depth[k];
    const uint8_t prev = k > first ? a.tok[k - 1] : T_NONE;
    const uint8_t next = k < last ? a.tok[k + 1] : T_NONE;
    bool ok;
    if (k == first) {
        ok = c == T_LP && d == 0 && next == T_LP;
    } else if (d < 1) {
        ok = false;
    } else if (c == T_LP) {
        ok = (d == 1 && (prev == T_LP || prev == T_CM) && next == T_LP) ||
             (d == 2 && prev == T_LP && next == T_NUM);
    } else if (c == T_RP) {
        ok = (d == 3 && prev == T_NUM && next == T_RP) ||
             (d == 2 && prev == T_RP && (next == T_CM || next == T_RP)) || (d == 1 && prev == T_RP && k == last);
    } else if (c == T_CM) {
        ok = (d == 3 && prev == T_NUM && next == T_NUM) || (d == 1 && prev == T_RP && next == T_LP);
    } else {  // number
        ok = d == 3;
        if (ok && prev != T_NUM) {
            ok = (prev == T_LP || prev == T_CM) && k + 3 <= last && a.tok[k + 1] == T_NUM &&
                 a.tok[k + 2] == T_NUM && (a.tok[k + 3] == T_CM || a.tok[k + 3] == T_RP);
        }
    }
    if (!ok) atomicMin(a.err_lit, L);
    a.ring_open[k] = c == T_LP && d == 2;
}

__global__ void literal_check_kernel(const uint32_t* lit_tok0, uint32_t n_lit, unsigned int* err_lit) {
    const uint32_t L = blockIdx.x * blockDim.x + threadIdx.x;
    if (L < n_lit && lit_tok0[L] == lit_tok0[L + 1]) atomicMin(err_lit, L);  // no tokens
}

__global__ void ring_index_kernel(const uint8_t* tok, const int* depth, const uint32_t* ring, const uint32_t* tok_num,
                                  uint32_t T, uint32_t* ring_n0, uint32_t* ring_n1, uint32_t* ring_tok) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= T) return;
    if (tok[k] == T_LP && depth[k] == 2) {
        ring_n0[ring[k]] = tok_num[k];
        ring_tok[ring[k]] = k;
    } else if (tok[k] == T_RP && depth[k] == 3) {
        ring_n1[ring[k] - 1] = tok_num[k];
    }
}

// wkt.cpp:119-128 (>= 4 points, closed), :152-154 (TIN: a triangle)
__global__ void ring_check_kernel(uint32_t n_rings, const uint32_t* ring_n0, const uint32_t* ring_n1,
                                  const uint32_t* ring_tok, const uint32_t* lit_tok0, uint32_t n_lit,
                                  const uint8_t* lit_kind, const double* nums, uint32_t* tcnt,
                                  unsigned int* err_lit) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_rings) return;
    const uint32_t L = literal_of(lit_tok0, n_lit, ring_tok[r]);
    const uint32_t n0 = ring_n0[r], n1 = ring_n1[r];
    const uint32_t P = (n1 - n0) / 3;
    bool ok = P >= 4;
    if (ok) {
        const double* f = nums + n0;
        const double* b = nums + n1 - 3;
        ok = f[0] == b[0] && f[1] == b[1] && f[2] == b[2];
    }
    if (ok && lit_kind[L] == 0) ok = P == 4;
    if (!ok) atomicMin(err_lit, L);
    tcnt[r] = ok ? P - 3 : 0;
}

// fan from the ring's first vertex (wkt.cpp:134-138): (p0, p_i, p_{i+1})
__global__ void emit_kernel(uint32_t n_rings, const uint32_t* ring_n0, const uint32_t* tcnt, const uint32_t* toff,
                            const double* nums, double* tri9) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n_rings) return;
    const double* p = nums + ring_n0[r];
    double* o = tri9 + 9ull * toff[r];
    for (uint32_t i = 1; i <= tcnt[r]; ++i, o += 9) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            o[c] = p[c];
            o[3 + c] = p[3 * i + c];
            o[6 + c] = p[3 * (i + 1) + c];
        }
    }
}

__global__ void face_offsets_kernel(uint32_t n_lit, const uint32_t* lit_tok0, const uint32_t* ring, uint32_t n_rings,
                                    const uint32_t* toff, uint64_t* off) {
    const uint32_t L = blockIdx.x * blockDim.x + threadIdx.x;
    if (L > n_lit) return;
    if (L == n_lit) {
        off[L] = toff[n_rings];
        return;
    }
    const uint32_t r0 = ring[lit_tok0[L]];  // rings before the literal's first token
    off[L] = toff[min(r0, n_rings)];
}

template <class T>
T* dnew(uint64_t n, cudaStream_t st) {
    T* p = nullptr;
    CK(cudaMallocAsync(&p, std::max<uint64_t>(1, n) * sizeof(T), st));
    return p;
}

struct Frees {
    cudaStream_t st;
    std::vector<void*> ptrs;
    template <class T>
    T* take(T* p) {
        ptrs.push_back(p);
        return p;
    }
    ~Frees() {
        for (void* p : ptrs) cudaFreeAsync(p, st);
    }
};

template <class F>
void cub_run(F&& f, cudaStream_t st, Frees& fr) {
    size_t bytes = 0;
    CK(f(nullptr, bytes));
    void* tmp = fr.take(dnew<char>(bytes, st));
    CK(f(tmp, bytes));
}

// ---- host: headers and the reference's error wording ----------------------
bool ieq(std::string_view a, std::string_view b) {
    if (a.size() != b.size()) return false;
    for (size_t i = 0; i < a.size(); ++i)
        if (std::tolower((unsigned char)a[i]) != std::tolower((unsigned char)b[i])) return false;
    return true;
}

struct Reader {  // byte cursor with the reference's token conventions
    std::string_view s;
    size_t p = 0;
    void ws() {
        while (p < s.size() && std::isspace((unsigned char)s[p])) ++p;
    }
    std::string_view word() {
        ws();
        const size_t b = p;
        while (p < s.size() && (std::isalpha((unsigned char)s[p]) || s[p] == '_')) ++p;
        return s.substr(b, p - b);
    }
};

struct Explain {  // first WktParseError of one literal, worded as wkt.cpp
    std::string what;
    uint64_t pos = 0;
};

struct ExplainFail {
    std::string msg;
    size_t pos;
};

class Explainer {
  public:
    explicit Explainer(std::string_view s) { R.s = s; }

    // Runs the reference grammar; returns false (and the error) on the first
    // violation, true when the literal is a valid geometry (kind in *kind:
    // 0 point, 1 line string, 2 mesh).
    bool run(Explain* e, int* kind) {
        try {
            top(kind);
            return true;
        } catch (const ExplainFail& f) {
            e->what = f.msg + " at position " + std::to_string(f.pos);
            e->pos = f.pos;
            return false;
        }
    }

  private:
    Reader R;
    [[noreturn]] static void fail(std::string m, size_t at) { throw ExplainFail{std::move(m), at}; }
    char peek() {
        R.ws();
        return R.p < R.s.size() ? R.s[R.p] : '\0';
    }
    void need(char c) {
        R.ws();
        if (R.p >= R.s.size() || R.s[R.p] != c) fail(std::string("expected '") + c + "'", R.p);
        ++R.p;
    }
    bool take(char c) {
        if (peek() != c || R.p >= R.s.size()) return false;
        ++R.p;
        return true;
    }
    double number() {
        R.ws();
        const size_t at = R.p;
        if (R.p < R.s.size() && std::isalpha((unsigned char)R.s[R.p])) {
            const std::string_view w = R.word();
            fail(ieq(w, "nan") || ieq(w, "inf") || ieq(w, "infinity") ? "non-finite coordinate" : "expected number",
                 at);
        }
        double v = 0.0;
        const char* b = R.s.data() + R.p;
        const auto res = std::from_chars(b, R.s.data() + R.s.size(), v);
        if (res.ec == std::errc::result_out_of_range) fail("non-finite coordinate", at);
        if (res.ec != std::errc() || res.ptr == b) fail("expected number", at);
        R.p = (size_t)(res.ptr - R.s.data());
        if (!std::isfinite(v)) fail("non-finite coordinate", at);
        return v;
    }
    struct P3 {
        double x, y, z;
        bool operator==(const P3& o) const { return x == o.x && y == o.y && z == o.z; }
    };
    P3 point() {
        const size_t at = R.p;
        P3 q;
        q.x = number();
        R.ws();
        if (R.p >= R.s.size() || R.s[R.p] == ',' || R.s[R.p] == ')') fail("incomplete coordinate triple", at);
        q.y = number();
        R.ws();
        if (R.p >= R.s.size() || R.s[R.p] == ',' || R.s[R.p] == ')')
            fail("expected Z coordinate (2D input not accepted)", R.p);
        q.z = number();
        return q;
    }
    std::vector<P3> points() {
        std::vector<P3> v;
        need('(');
        do v.push_back(point());
        while (take(','));
        need(')');
        return v;
    }
    size_t ring() {
        need('(');
        const size_t at = R.p;
        std::vector<P3> v = points();
        if (peek() == ',') fail("interior rings are not supported", R.p);
        need(')');
        if (v.size() < 4) fail("polygon ring must have at least 4 points including closure", at);
        if (!(v.front() == v.back())) fail("polygon ring is not closed (first point != last point)", at);
        return v.size() - 1;
    }
    void surface(bool tin) {
        need('(');
        do {
            const size_t at = R.p;
            const size_t n = ring();
            if (tin && n != 3) fail("TIN patch must be a triangle (4 points including closure)", at);
        } while (take(','));
        need(')');
    }
    void zmark() {
        const size_t at = R.p;
        R.ws();
        const std::string_view w = R.word();
        if (w.empty()) fail("expected 'Z' dimension marker (2D input not accepted)", at);
        if (ieq(w, "ZM") || ieq(w, "M")) fail("measured coordinates are not supported", at);
        if (!ieq(w, "Z")) fail("expected 'Z' dimension marker", at);
    }
    void top(int* kind) {
        R.ws();
        const size_t at = R.p;
        const std::string_view kw = R.word();
        if (kw.empty()) fail("empty WKT input", at);
        if (ieq(kw, "POINT")) {
            zmark();
            need('(');
            point();
            need(')');
            *kind = 0;
        } else if (ieq(kw, "LINESTRING")) {
            zmark();
            const size_t ls = R.p;
            if (points().size() < 2) fail("LINESTRING requires at least 2 points", ls);
            *kind = 1;
        } else if (ieq(kw, "TIN") || ieq(kw, "POLYHEDRALSURFACE")) {
            zmark();
            surface(ieq(kw, "TIN"));
            *kind = 2;
        } else {
            fail("unknown geometry type '" + std::string(kw) + "'", at);
        }
        R.ws();
        if (R.p < R.s.size()) fail("trailing input after geometry", R.p);
    }
};

[[noreturn]] void throw_literal(const char* text, const uint64_t* lit_off, uint64_t L, const char* fallback) {
    Explain e;
    int kind = -1;
    const std::string_view s(text + lit_off[L], lit_off[L + 1] - lit_off[L]);
    if (Explainer(s).run(&e, &kind)) {
        if (kind != 2) throw WktError("WKT geometry is not a mesh (TIN Z / POLYHEDRALSURFACE Z expected)", L, 0);
        throw CudaError(std::string("internal: device WKT parser rejected a valid literal (") + fallback + ")");
    }
    throw WktError(e.what, L, e.pos);
}

// Header of literal L: kind (0 TIN, 1 POLYHEDRALSURFACE) and where its body
// starts; false when the header is not a mesh header.
bool header(std::string_view s, uint8_t* kind, size_t* body) {
    Reader r{s};
    const std::string_view kw = r.word();
    if (ieq(kw, "TIN")) *kind = 0;
    else if (ieq(kw, "POLYHEDRALSURFACE")) *kind = 1;
    else return false;
    if (!ieq(r.word(), "Z")) return false;
    *body = r.p;
    return true;
}

struct BatchOut {
    double* tri9 = nullptr;  // device, n_tris x 9
    uint64_t n_tris = 0;
    std::vector<uint64_t> faces;  // per literal
};

// Parses literals [L0, L1) (their text is text[lit_off[L0], lit_off[L1])).
void parse_batch(const char* text, const uint64_t* lit_off, uint64_t L0, uint64_t L1, cudaStream_t st, BatchOut* out) {
    const uint32_t n_lit = (uint32_t)(L1 - L0);
    const uint64_t base = lit_off[L0], n = lit_off[L1] - base;
    std::vector<uint64_t> bb(n_lit), be(n_lit);
    std::vector<uint8_t> kind(n_lit);
    for (uint32_t i = 0; i < n_lit; ++i) {
        const uint64_t L = L0 + i;
        size_t body = 0;
        const std::string_view s(text + lit_off[L], lit_off[L + 1] - lit_off[L]);
        if (!header(s, &kind[i], &body)) throw_literal(text, lit_off, L, "header");
        bb[i] = lit_off[L] - base + body;
        be[i] = lit_off[L + 1] - base;
        if (bb[i] == be[i]) throw_literal(text, lit_off, L, "empty body");
    }
    Frees fr{st, {}};
    char* d_text_buf = fr.take(dnew<char>(kTextPad + n + kLexChunk + kLexHalo + 16, st));
    char* d_text = d_text_buf + kTextPad;
    CK(cudaMemsetAsync(d_text_buf, 0, kTextPad, st));
    CK(cudaMemsetAsync(d_text + n, 0, kLexChunk + kLexHalo + 16, st));
    uint64_t* d_bb = fr.take(dnew<uint64_t>(n_lit, st));
    uint64_t* d_be = fr.take(dnew<uint64_t>(n_lit, st));
    uint8_t* d_kind = fr.take(dnew<uint8_t>(n_lit, st));
    h2d(d_text, text + base, n, st);
    CK(cudaMemcpyAsync(d_bb, bb.data(), n_lit * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_be, be.data(), n_lit * sizeof(uint64_t), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(d_kind, kind.data(), n_lit, cudaMemcpyHostToDevice, st));

    const uint64_t nthr = (n + kSpan - 1) / kSpan;
    uint32_t* cnt = fr.take(dnew<uint32_t>(2 * (nthr + 1), st));  // tokens | numbers
    uint32_t* off = fr.take(dnew<uint32_t>(2 * (nthr + 1), st));
    unsigned long long* err_byte = fr.take(dnew<unsigned long long>(1, st));
    unsigned int* err_lit = fr.take(dnew<unsigned int>(2, st));  // literal, slow count
    CK(cudaMemsetAsync(cnt, 0, 2 * (nthr + 1) * sizeof(uint32_t), st));
    CK(cudaMemsetAsync(err_byte, 0xff, sizeof(unsigned long long), st));
    CK(cudaMemsetAsync(err_lit, 0xff, sizeof(unsigned int), st));
    CK(cudaMemsetAsync(err_lit + 1, 0, sizeof(unsigned int), st));

    LexArgs a{};
    a.text = d_text;
    a.n = n;
    a.bb = d_bb;
    a.be = d_be;
    a.n_lit = n_lit;
    a.err_byte = err_byte;
    a.n_slow = err_lit + 1;
    a.cnt_tok = cnt;
    a.cnt_num = cnt + nthr + 1;
    a.span_multi = fr.take(dnew<uint8_t>(nthr, st));
    const unsigned lex_blocks = (unsigned)((nthr + kLexThreads - 1) / kLexThreads);
    lex_kernel<0><<<lex_blocks, kLexThreads, 0, st>>>(a);
    CK(cudaGetLastError());
    const int items = (int)(nthr + 1);
    for (int h = 0; h < 2; ++h)
        cub_run([&](void* tmp, size_t& bytes) {
            return cub::DeviceScan::ExclusiveSum(tmp, bytes, cnt + h * (nthr + 1), off + h * (nthr + 1), items, st);
        }, st, fr);
    uint32_t T = 0, NN = 0;
    unsigned long long eb = 0;
    CK(cudaMemcpyAsync(&T, off + nthr, sizeof T, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&NN, off + 2 * nthr + 1, sizeof NN, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&eb, err_byte, sizeof eb, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (eb != ~0ull) {  // a lexical error: the literal holding that byte
        const uint64_t at = eb + base;
        uint64_t L = L0;
        while (L + 1 < L1 && lit_off[L + 1] <= at) ++L;
        throw_literal(text, lit_off, L, "lexer");
    }

    uint8_t* tok = fr.take(dnew<uint8_t>(T, st));
    uint32_t* tok_num = fr.take(dnew<uint32_t>(T, st));
    double* nums = fr.take(dnew<double>(NN, st));
    uint32_t* slow = fr.take(dnew<uint32_t>(NN, st));
    uint64_t* slow_pos = fr.take(dnew<uint64_t>(NN, st));
    uint32_t* slow_len = fr.take(dnew<uint32_t>(NN, st));
    uint32_t* lit_tok0 = fr.take(dnew<uint32_t>(n_lit + 1, st));
    CK(cudaMemsetAsync(lit_tok0, 0xff, (n_lit + 1) * sizeof(uint32_t), st));
    CK(cudaMemcpyAsync(lit_tok0 + n_lit, &T, sizeof T, cudaMemcpyHostToDevice, st));
    a.cnt_tok = off;
    a.cnt_num = off + nthr + 1;
    a.tok = tok;
    a.tok_num = tok_num;
    a.nums = nums;
    a.slow = slow;
    a.slow_pos = slow_pos;
    a.slow_len = slow_len;
    a.lit_tok0 = lit_tok0;
    lex_kernel<1><<<lex_blocks, kLexThreads, 0, st>>>(a);
    CK(cudaGetLastError());
    if (NN) {
        slow_number_kernel<<<(unsigned)((NN + 127) / 128), 128, 0, st>>>(d_text, slow, slow_pos, slow_len, err_lit + 1,
                                                                          nums, err_byte);
        CK(cudaGetLastError());
    }

    // grammar
    int* depth = fr.take(dnew<int>(T + 1, st));
    uint32_t* ring_open = fr.take(dnew<uint32_t>(T + 1, st));
    uint32_t* ring = fr.take(dnew<uint32_t>(T + 1, st));
    CK(cudaMemsetAsync(ring_open + T, 0, sizeof(uint32_t), st));
    if (T) {
        cub::TransformInputIterator<int, DepthDelta, const uint8_t*> dd(tok, DepthDelta{});
        cub_run([&](void* tmp, size_t& bytes) {
            return cub::DeviceScan::ExclusiveSum(tmp, bytes, dd, depth, (int)T, st);
        }, st, fr);
        GramArgs g{tok, depth, T, lit_tok0, n_lit, ring_open, err_lit};
        grammar_kernel<<<(T + 255) / 256, 256, 0, st>>>(g);
        CK(cudaGetLastError());
    }
    literal_check_kernel<<<(n_lit + 255) / 256, 256, 0, st>>>(lit_tok0, n_lit, err_lit);
    CK(cudaGetLastError());
    cub_run([&](void* tmp, size_t& bytes) {
        return cub::DeviceScan::ExclusiveSum(tmp, bytes, ring_open, ring, (int)(T + 1), st);
    }, st, fr);
    uint32_t n_rings = 0, el = 0;
    CK(cudaMemcpyAsync(&n_rings, ring + T, sizeof n_rings, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&el, err_lit, sizeof el, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&eb, err_byte, sizeof eb, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    uint64_t bad = ~0ull;
    if (el != ~0u) bad = L0 + el;
    if (eb != ~0ull) {  // a hard number out of range
        const uint64_t at = eb + base;
        uint64_t L = L0;
        while (L + 1 < L1 && lit_off[L + 1] <= at) ++L;
        bad = std::min(bad, L);
    }
    if (bad != ~0ull) throw_literal(text, lit_off, bad, "grammar");

    // rings -> faces
    uint32_t* ring_n0 = fr.take(dnew<uint32_t>(n_rings, st));
    uint32_t* ring_n1 = fr.take(dnew<uint32_t>(n_rings, st));
    uint32_t* ring_tok = fr.take(dnew<uint32_t>(n_rings, st));
    uint32_t* tcnt = fr.take(dnew<uint32_t>(n_rings + 1, st));
    uint32_t* toff = fr.take(dnew<uint32_t>(n_rings + 1, st));
    CK(cudaMemsetAsync(tcnt + n_rings, 0, sizeof(uint32_t), st));
    if (n_rings) {
        ring_index_kernel<<<(T + 255) / 256, 256, 0, st>>>(tok, depth, ring, tok_num, T, ring_n0, ring_n1, ring_tok);
        CK(cudaGetLastError());
        ring_check_kernel<<<(n_rings + 255) / 256, 256, 0, st>>>(n_rings, ring_n0, ring_n1, ring_tok, lit_tok0, n_lit,
                                                                 d_kind, nums, tcnt, err_lit);
        CK(cudaGetLastError());
    }
    cub_run([&](void* tmp, size_t& bytes) {
        return cub::DeviceScan::ExclusiveSum(tmp, bytes, tcnt, toff, (int)(n_rings + 1), st);
    }, st, fr);
    uint32_t n_tris = 0;
    CK(cudaMemcpyAsync(&n_tris, toff + n_rings, sizeof n_tris, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&el, err_lit, sizeof el, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (el != ~0u) throw_literal(text, lit_off, L0 + el, "rings");

    out->n_tris = n_tris;
    out->tri9 = dnew<double>(9ull * n_tris, st);
    uint64_t* d_foff = fr.take(dnew<uint64_t>(n_lit + 1, st));
    if (n_rings) {
        emit_kernel<<<(n_rings + 127) / 128, 128, 0, st>>>(n_rings, ring_n0, tcnt, toff, nums, out->tri9);
        CK(cudaGetLastError());
    }
    face_offsets_kernel<<<(n_lit + 1 + 255) / 256, 256, 0, st>>>(n_lit, lit_tok0, ring, n_rings, toff, d_foff);
    CK(cudaGetLastError());
    std::vector<uint64_t> foff(n_lit + 1);
    CK(cudaMemcpyAsync(foff.data(), d_foff, (n_lit + 1) * sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    out->faces.resize(n_lit);
    for (uint32_t i = 0; i < n_lit; ++i) out->faces[i] = foff[i + 1] - foff[i];
}

}  // namespace

void wkt_build(Geom* g, const char* text, const uint64_t* lit_off, uint64_t n_lit, cudaStream_t st) {
    if (n_lit == 0) throw std::invalid_argument("no WKT literals");
    for (uint64_t L = 0; L < n_lit; ++L) {
        if (lit_off[L + 1] < lit_off[L]) throw std::invalid_argument("literal offsets must be non-decreasing");
        if (lit_off[L + 1] - lit_off[L] > kBatchBytes) throw std::invalid_argument("WKT literal larger than 2 GiB");
    }
    std::vector<BatchOut> parts;
    try {
        for (uint64_t L0 = 0; L0 < n_lit;) {
            uint64_t L1 = L0 + 1;
            while (L1 < n_lit && lit_off[L1 + 1] - lit_off[L0] <= kBatchBytes && L1 - L0 < (1ull << 30)) ++L1;
            parts.emplace_back();
            parse_batch(text, lit_off, L0, L1, st, &parts.back());
            L0 = L1;
        }
        std::vector<uint64_t> off(n_lit + 1, 0);
        uint64_t total = 0, L = 0;
        for (const BatchOut& b : parts) {
            for (uint64_t f : b.faces) off[L + 1] = off[L] + f, ++L;
            total += b.n_tris;
        }
        double* tri9 = nullptr;
        if (parts.size() == 1) {
            tri9 = parts[0].tri9;
            parts[0].tri9 = nullptr;
        } else {
            tri9 = dnew<double>(9 * total, st);
            uint64_t at = 0;
            for (BatchOut& b : parts) {
                CK(cudaMemcpyAsync(tri9 + 9 * at, b.tri9, 9 * b.n_tris * sizeof(double), cudaMemcpyDeviceToDevice, st));
                at += b.n_tris;
            }
        }
        try {
            geom_build(g, tri9, total, off.data(), n_lit, st, true);
        } catch (...) {
            cudaFreeAsync(tri9, st);
            throw;
        }
        CK(cudaFreeAsync(tri9, st));
    } catch (...) {
        for (BatchOut& b : parts)
            if (b.tri9) cudaFreeAsync(b.tri9, st);
        throw;
    }
    for (BatchOut& b : parts)
        if (b.tri9) CK(cudaFreeAsync(b.tri9, st));
}

// Device planes -> host AoS (face order), the store's inverse.
__global__ void download_kernel(const double* planes, uint64_t n, uint64_t n_pad, double* out) {
    const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
#pragma unroll
    for (int c = 0; c < 9; ++c) out[9 * i + c] = planes[(uint64_t)(F_V + c) * n_pad + i];
}

void geom_download(const Geom& g, double* host_tri9, cudaStream_t st) {
    if (!g.n) return;
    double* d = dnew<double>(9 * g.n, st);
    download_kernel<<<(unsigned)((g.n + 255) / 256), 256, 0, st>>>(g.planes, g.n, g.n_pad, d);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) {
        try {
            d2h(host_tri9, d, 9 * g.n * sizeof(double), st);
        } catch (...) {
            cudaFreeAsync(d, st);
            throw;
        }
    }
    cudaFreeAsync(d, st);
    CK(e);
    CK(cudaStreamSynchronize(st));
}

}  // namespace tdb

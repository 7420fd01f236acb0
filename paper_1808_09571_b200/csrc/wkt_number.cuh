// Decimal text -> binary64, bit-identical to std::from_chars(first, last,
// double&) as the reference's WKT reader calls it (wkt.cpp:84-95): syntax
// `-? (digits (. digits?)? | . digits) ([eE] [+-]? digits)?` with maximal
// munch (an exponent is consumed only when digits follow), correctly rounded
// to nearest-even; `result_out_of_range` when the value overflows to
// infinity or a nonzero value rounds to zero (the reference turns both into
// "non-finite coordinate").
//
// Three tiers, each exact where it answers:
//   1. Eisel-Lemire over the first 19 significant digits with the 128-bit
//      truncated powers of ten (pow10_table.h); for longer inputs the answer
//      is accepted only when mantissa and mantissa+1 round alike;
//   2. otherwise `slow` — a big-integer comparison of the full digit string
//      against the halfway points around a candidate (parse_number_slow),
//      run by a separate pass on the rare tokens that need it.
// Compiled as device code in wkt.cu and as host code in the CPU fuzz test
// (tests/cpp/number_test.cpp), which checks it against std::from_chars.
#pragma once

#include <cstdint>

#include "pow10_table.h"

#ifdef __CUDACC__
#define TDB_NUM_FN __device__ __forceinline__
#define TDB_NUM_NOINLINE __device__ __noinline__
#else
#define TDB_NUM_FN inline
#define TDB_NUM_NOINLINE inline
#endif

namespace tdb {
namespace num {

enum Status : int { kOk = 0, kNoMatch = 1, kRange = 2, kSlow = 3 };

struct Scan {
    int status;
    uint32_t len;  // bytes consumed (kOk, kRange, kSlow)
    double value;  // kOk
};

TDB_NUM_FN bool is_digit(char c) { return c >= '0' && c <= '9'; }

TDB_NUM_FN int clz64(uint64_t x) {
#ifdef __CUDA_ARCH__
    return __clzll((long long)x);
#else
    return __builtin_clzll(x);
#endif
}

TDB_NUM_FN void mul64(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
#ifdef __CUDA_ARCH__
    lo = a * b;
    hi = __umul64hi(a, b);
#else
    const unsigned __int128 p = (unsigned __int128)a * b;
    lo = (uint64_t)p;
    hi = (uint64_t)(p >> 64);
#endif
}

TDB_NUM_FN double from_bits(uint64_t b) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double((long long)b);
#else
    double d;
    __builtin_memcpy(&d, &b, 8);
    return d;
#endif
}

TDB_NUM_FN uint64_t to_bits(double d) {
#ifdef __CUDA_ARCH__
    return (uint64_t)__double_as_longlong(d);
#else
    uint64_t b;
    __builtin_memcpy(&b, &d, 8);
    return b;
#endif
}

// Eisel-Lemire: w * 10^q (w != 0) as a positive binary64's bits; false when
// the 128-bit product cannot decide the rounding, or the result is subnormal
// or overflows (all left to the slow tier).
TDB_NUM_FN bool eisel_lemire(uint64_t w, int q, uint64_t& bits) {
    if (q < kPow10Min || q > kPow10Max) return false;
    const uint64_t* t = kPow10Mant[q - kPow10Min];
    const int lz = clz64(w);
    w <<= lz;
    uint64_t e2 = (uint64_t)(((217706 * q) >> 16) + 64 + 1023) - (uint64_t)lz;
    uint64_t hi, lo;
    mul64(w, t[0], hi, lo);
    if ((hi & 0x1FF) == 0x1FF && lo + w < w) {  // widen with the low 64 bits of 10^q
        uint64_t yhi, ylo;
        mul64(w, t[1], yhi, ylo);
        uint64_t mhi = hi, mlo = lo + yhi;
        if (mlo < lo) ++mhi;
        if ((mhi & 0x1FF) == 0x1FF && mlo + 1 == 0 && ylo + w < w) return false;
        hi = mhi, lo = mlo;
    }
    const uint64_t msb = hi >> 63;
    uint64_t m = hi >> (msb + 9);
    e2 -= 1 ^ msb;
    if (lo == 0 && (hi & 0x1FF) == 0 && (m & 3) == 1) return false;  // halfway ambiguity
    m += m & 1;
    m >>= 1;
    if (m >> 53) {
        m >>= 1;
        ++e2;
    }
    if (e2 - 1 >= 0x7FF - 1) return false;  // subnormal or overflow
    bits = (e2 << 52) | (m & 0x000FFFFFFFFFFFFFull);
    return true;
}

// Fast tier over [s, end): syntax, 19-digit mantissa, Eisel-Lemire.
// kValue = false scans the syntax only (token counting): the status is then
// kOk for every in-range number, kRange only for the gross range cases.
template <bool kValue = true>
TDB_NUM_FN Scan parse_number(const char* s, const char* end) {
    const char* p = s;
    const bool neg = p < end && *p == '-';
    if (neg) ++p;
    uint64_t w = 0;
    int nd = 0;            // significant digits kept in w
    long long e10 = 0;     // value = w * 10^e10 (before the exponent part)
    bool trunc = false, any = false;
    while (p < end && is_digit(*p)) {
        const int d = *p - '0';
        any = true;
        if (w == 0 && d == 0 && nd == 0) {
        } else if (nd < 19) {
            w = w * 10 + (uint64_t)d;
            ++nd;
        } else {
            ++e10;
            trunc |= d != 0;
        }
        ++p;
    }
    if (p < end && *p == '.') {
        const char* f = p + 1;
        const char* q = f;
        while (q < end && is_digit(*q)) {
            const int d = *q - '0';
            if (w == 0 && d == 0 && nd == 0) {
                --e10;
            } else if (nd < 19) {
                w = w * 10 + (uint64_t)d;
                ++nd;
                --e10;
            } else {
                trunc |= d != 0;
            }
            ++q;
        }
        if (q > f) any = true;
        if (any) p = q;  // "1." consumes the point; "." alone is no match
    }
    if (!any) return Scan{kNoMatch, 0, 0.0};
    if (p < end && (*p == 'e' || *p == 'E')) {
        const char* q = p + 1;
        bool eneg = false;
        if (q < end && (*q == '+' || *q == '-')) eneg = *q++ == '-';
        if (q < end && is_digit(*q)) {
            long long ev = 0;
            while (q < end && is_digit(*q)) {
                if (ev < 100000000) ev = ev * 10 + (*q - '0');
                ++q;
            }
            e10 += eneg ? -ev : ev;
            p = q;
        }
    }
    const uint32_t len = (uint32_t)(p - s);
    if (w == 0) return Scan{kOk, len, neg ? -0.0 : 0.0};
    // decimal exponent of the leading digit: e10 + nd - 1
    const long long top = e10 + nd - 1;
    if (top >= 309) return Scan{kRange, len, 0.0};   // >= 1e309 > DBL_MAX
    if (top < -325) return Scan{kRange, len, 0.0};   // < 1e-325 < 2^-1075: rounds to 0
    if (!kValue) return Scan{kOk, len, 0.0};
    uint64_t b;
    if (eisel_lemire(w, (int)e10, b)) {
        if (trunc) {
            uint64_t b2;
            if (!eisel_lemire(w + 1, (int)e10, b2) || b2 != b) return Scan{kSlow, len, 0.0};
        }
        return Scan{kOk, len, from_bits(b | (neg ? 0x8000000000000000ull : 0ull))};
    }
    return Scan{kSlow, len, 0.0};
}

// ---- slow tier: big-integer comparison --------------------------------------
constexpr int kBigLimbs = 140;    // 4480 bits
constexpr int kMaxDigits = 800;   // significant digits kept; the rest is a sticky bit

struct Big {
    uint32_t l[kBigLimbs];
    int n;  // limbs in use
};

TDB_NUM_FN void big_set(Big& a, uint64_t v) {
    a.n = 0;
    while (v) {
        a.l[a.n++] = (uint32_t)v;
        v >>= 32;
    }
}

TDB_NUM_FN void big_mul_small(Big& a, uint32_t m, uint32_t add = 0) {
    uint64_t carry = add;
    for (int i = 0; i < a.n; ++i) {
        const uint64_t t = (uint64_t)a.l[i] * m + carry;
        a.l[i] = (uint32_t)t;
        carry = t >> 32;
    }
    if (carry && a.n < kBigLimbs) a.l[a.n++] = (uint32_t)carry;
}

TDB_NUM_FN void big_mul_pow5(Big& a, long long k) {
    while (k >= 13) {
        big_mul_small(a, 1220703125u);  // 5^13
        k -= 13;
    }
    uint32_t r = 1;
    while (k-- > 0) r *= 5;
    if (r > 1) big_mul_small(a, r);
}

TDB_NUM_FN void big_shl(Big& a, long long s) {
    if (a.n == 0 || s <= 0) return;
    const int w = (int)(s >> 5), b = (int)(s & 31);
    int n = a.n + w + 1;
    if (n > kBigLimbs) n = kBigLimbs;
    for (int i = n - 1; i >= 0; --i) {
        const int src = i - w;
        uint32_t hi = src >= 0 && src < a.n ? a.l[src] : 0u;
        uint32_t lo = src - 1 >= 0 && src - 1 < a.n ? a.l[src - 1] : 0u;
        a.l[i] = b ? (hi << b) | (lo >> (32 - b)) : hi;
    }
    a.n = n;
    while (a.n && a.l[a.n - 1] == 0) --a.n;
}

TDB_NUM_FN int big_cmp(const Big& a, const Big& b) {
    if (a.n != b.n) return a.n < b.n ? -1 : 1;
    for (int i = a.n - 1; i >= 0; --i)
        if (a.l[i] != b.l[i]) return a.l[i] < b.l[i] ? -1 : 1;
    return 0;
}

// sign(D * 10^e10 - h * 2^e2), D given as a big integer
TDB_NUM_FN int cmp_scaled(const Big& D, long long e10, uint64_t h, long long e2, Big& L, Big& R) {
    L = D;
    big_set(R, h);
    if (e10 >= 0) {
        big_mul_pow5(L, e10);
    } else {
        big_mul_pow5(R, -e10);
    }
    // remaining binary factors: L * 2^e10 vs R * 2^e2
    if (e10 > e2) big_shl(L, e10 - e2);
    else big_shl(R, e2 - e10);
    return big_cmp(L, R);
}

// halfway point above the non-negative finite double with bits `b`:
// (2m + 1) * 2^(E - 1)
TDB_NUM_FN void halfway_up(uint64_t b, uint64_t& h, long long& e2) {
    const uint64_t ex = b >> 52, fr = b & 0x000FFFFFFFFFFFFFull;
    uint64_t m;
    long long E;
    if (ex == 0) {
        m = fr;
        E = -1074;
    } else {
        m = fr | (1ull << 52);
        E = (long long)ex - 1075;
    }
    h = 2 * m + 1;
    e2 = E - 1;
}

// Slow tier: the correctly rounded value of [s, s+len) (a token the fast
// tier scanned as kSlow). Returns kOk or kRange.
TDB_NUM_NOINLINE Scan parse_number_slow(const char* s, uint32_t len) {
    const char* p = s;
    const char* end = s + len;
    const bool neg = *p == '-';
    if (neg) ++p;
    Big D;
    D.n = 0;
    int nd = 0;
    long long e10 = 0;
    bool sticky = false;
    uint32_t chunk = 0, chunk_mul = 1;
    auto push = [&](int d) {
        chunk = chunk * 10 + (uint32_t)d;
        chunk_mul *= 10;
        if (chunk_mul == 1000000000u) {
            big_mul_small(D, chunk_mul, chunk);
            chunk = 0, chunk_mul = 1;
        }
    };
    bool frac = false;
    for (; p < end; ++p) {
        const char c = *p;
        if (c == '.') {
            frac = true;
            continue;
        }
        if (!is_digit(c)) break;
        const int d = c - '0';
        if (nd == 0 && d == 0) {
            if (frac) --e10;
            continue;
        }
        if (nd < kMaxDigits) {
            push(d);
            ++nd;
            if (frac) --e10;
        } else {
            sticky |= d != 0;
            if (!frac) ++e10;
        }
    }
    if (chunk_mul > 1) big_mul_small(D, chunk_mul, chunk);
    if (p < end && (*p == 'e' || *p == 'E')) {
        ++p;
        bool eneg = false;
        if (*p == '+' || *p == '-') eneg = *p++ == '-';
        long long ev = 0;
        for (; p < end && is_digit(*p); ++p)
            if (ev < 100000000) ev = ev * 10 + (*p - '0');
        e10 += eneg ? -ev : ev;
    }
    if (D.n == 0) return Scan{kOk, len, neg ? -0.0 : 0.0};
    const long long top = e10 + nd - 1;
    if (top >= 309 || top < -325) return Scan{kRange, len, 0.0};

    // candidate: the leading 19 digits scaled in binary64 (a few ulps off)
    double c;
    {
        uint64_t w = 0;
        int k = 0;
        long long ew = e10 + (nd > 19 ? nd - 19 : 0);
        // re-read the leading digits
        const char* r = neg ? s + 1 : s;
        for (; r < end && k < 19; ++r) {
            if (*r == '.') continue;
            if (!is_digit(*r)) break;
            const int d = *r - '0';
            if (k == 0 && d == 0) continue;
            w = w * 10 + (uint64_t)d;
            ++k;
        }
        c = (double)w;
        const double p10[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,  1e8,  1e9,  1e10, 1e11,
                                1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};
        while (ew > 0) {
            const int s1 = ew > 22 ? 22 : (int)ew;
            c *= p10[s1];
            ew -= s1;
        }
        while (ew < 0) {
            const int s1 = -ew > 22 ? 22 : (int)-ew;
            c /= p10[s1];
            ew += s1;
        }
    }
    uint64_t b = to_bits(c);
    if (b >= 0x7FF0000000000000ull) b = 0x7FEFFFFFFFFFFFFFull;  // start from DBL_MAX
    Big L, R;
    for (int it = 0; it < 256; ++it) {
        uint64_t h;
        long long e2;
        halfway_up(b, h, e2);
        int r = cmp_scaled(D, e10, h, e2, L, R);
        if (r == 0 && sticky) r = 1;
        const bool odd = b & 1;
        if (r > 0 || (r == 0 && odd)) {  // above the upper halfway: next double
            ++b;
            if (b >= 0x7FF0000000000000ull) return Scan{kRange, len, 0.0};
            continue;
        }
        if (b > 0) {
            halfway_up(b - 1, h, e2);
            r = cmp_scaled(D, e10, h, e2, L, R);
            if (r == 0 && sticky) r = 1;
            if (r < 0 || (r == 0 && odd)) {
                --b;
                continue;
            }
        }
        break;
    }
    if (b == 0) return Scan{kRange, len, 0.0};  // a nonzero decimal that rounds to zero
    return Scan{kOk, len, from_bits(b | (neg ? 0x8000000000000000ull : 0ull))};
}

}  // namespace num
}  // namespace tdb

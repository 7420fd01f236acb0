// Host fuzz test: csrc/wkt_number.cuh (the device decimal parser, compiled
// here as host code) against std::from_chars, the reference WKT reader's
// number routine (wkt.cpp:84-95). Every case must agree on status, bytes
// consumed and the result's bits.
//   g++ -std=c++20 -O2 -I paper_1808_09571_b200/csrc tests/cpp/number_test.cpp
//   ./a.out [cases] [seed]
#include <charconv>
#include <cinttypes>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <system_error>

#include "wkt_number.cuh"

using namespace tdb::num;

static uint64_t bits_of(double d) {
    uint64_t b;
    std::memcpy(&b, &d, 8);
    return b;
}

static long n_cases = 0, n_slow = 0, n_fail = 0;

static void check(const std::string& s) {
    ++n_cases;
    double ref = 0.0;
    auto r = std::from_chars(s.data(), s.data() + s.size(), ref);
    Scan m = parse_number(s.data(), s.data() + s.size());
    if (m.status == kSlow) {
        ++n_slow;
        m = parse_number_slow(s.data(), m.len);
    }
    bool ok;
    if (r.ec == std::errc::invalid_argument) {
        ok = m.status == kNoMatch;
    } else if (r.ec == std::errc::result_out_of_range) {
        ok = m.status == kRange && m.len == (uint32_t)(r.ptr - s.data());
    } else {
        ok = m.status == kOk && m.len == (uint32_t)(r.ptr - s.data()) && bits_of(m.value) == bits_of(ref);
    }
    if (!ok) {
        if (++n_fail <= 20)
            std::printf("MISMATCH \"%.120s\"%s: ref ec=%d len=%ld bits=%016" PRIx64 " | ours st=%d len=%u bits=%016" PRIx64
                        "\n",
                        s.c_str(), s.size() > 120 ? "..." : "", (int)r.ec, (long)(r.ptr - s.data()), bits_of(ref),
                        m.status, m.len, bits_of(m.value));
    }
}

int main(int argc, char** argv) {
    const long cases = argc > 1 ? std::atol(argv[1]) : 200000;
    std::mt19937_64 rng(argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 42);
    auto u = [&](uint64_t n) { return rng() % n; };
    char buf[4096];

    // fixed syntax / range edge cases
    const char* fixed[] = {"0", "-0", "1", "-1", "1.", "-1.", ".5", "-.5", ".", "-", "-.", "--1", "+1", "1e", "1e+",
                           "1e-", "1E5", "1e+5", "1e-5", "1.e5", ".e5", "00012", "000.000", "0e999999999999",
                           "1e400", "1e-400", "4.9e-324", "2.4703282292062327e-324", "2.4703282292062328e-324",
                           "2.5e-324", "3e-324", "1e-320", "2.2250738585072011e-308", "2.2250738585072014e-308",
                           "1.7976931348623157e308", "1.7976931348623158e308", "1.7976931348623159e308",
                           "9007199254740993", "9007199254740992.5", "9007199254740993.0000000000000000001",
                           "123456789012345678901234567890", "1e-99999999999999", "1e99999999999999",
                           "0.1", "0.2", "0.3", "1e23", "8.5e-322", "1x", "1.5.5", "1-2", "7e-10e3",
                           "4.9406564584124654e-324", "2.47032822920623272088e-324",
                           "179769313486231580793728971405303415079934132710037826936173778980444968292764750946649017977587"
                           "207096330286416692887910946555547851940402630657488671505820681908902000708383676273854845817711"
                           "531764475730270069855571366959622842914819860834936475292719074168444365510704342711559699508093"
                           "0422968"};
    for (const char* f : fixed) check(f);

    // the exact decimal of the smallest subnormal halfway point (rounds to 0: out of range)
    {
        std::string h = "2.";
        long double x = 0x1p-1075L;
        std::snprintf(buf, sizeof buf, "%.800Le", x);
        check(buf);
        h = buf;
        h.insert(h.find('e'), "1");  // just above halfway: rounds up to 2^-1074
        check(h);
    }

    for (long i = 0; i < cases; ++i) {
        const int kind = (int)u(8);
        std::string s;
        if (kind == 0) {  // random double, shortest round trip
            double d;
            uint64_t b = rng() & 0x7FFFFFFFFFFFFFFFull;
            std::memcpy(&d, &b, 8);
            if (!std::isfinite(d)) continue;
            auto t = std::to_chars(buf, buf + sizeof buf, d);
            s.assign(buf, t.ptr);
        } else if (kind == 1) {  // random double, 1..25 significant digits
            double d;
            uint64_t b = rng() & 0x7FFFFFFFFFFFFFFFull;
            std::memcpy(&d, &b, 8);
            if (!std::isfinite(d)) continue;
            std::snprintf(buf, sizeof buf, "%.*e", (int)u(25), d);
            s = buf;
        } else if (kind == 2) {  // exact halfway between neighbours, +- a nudge
            double d;
            uint64_t b = (rng() % 0x7FEFFFFFFFFFFFFFull);
            std::memcpy(&d, &b, 8);
            const long double mid = ((long double)d + (long double)std::nextafter(d, INFINITY)) / 2;
            std::snprintf(buf, sizeof buf, "%.790Le", mid);
            s = buf;
            // trim trailing zeros of the mantissa to keep it exact but short
            const size_t e = s.find('e');
            size_t z = e;
            while (z > 0 && s[z - 1] == '0') --z;
            if (s[z - 1] == '.') --z;
            s = s.substr(0, z) + s.substr(e);
            const int nudge = (int)u(3);
            if (nudge == 1) {  // slightly above
                const size_t ee = s.find('e');
                s.insert(ee, s.find('.') == std::string::npos ? ".00000000000000000000001" : "00000000000000000001");
            } else if (nudge == 2) {  // drop the last digit: slightly below
                const size_t ee = s.find('e');
                if (ee > 3) s.erase(ee - 1, 1);
            }
        } else if (kind == 3) {  // random digit strings, random exponent
            const int nd = 1 + (int)u(u(4) == 0 ? 900 : 30);
            if (u(2)) s += '-';
            const int point = (int)u(nd + 1);
            for (int k = 0; k < nd; ++k) {
                if (k == point && u(2)) s += '.';
                s += (char)('0' + u(10));
            }
            if (u(3)) {
                s += u(2) ? 'e' : 'E';
                const int r = (int)u(3);
                if (r == 1) s += '-';
                if (r == 2) s += '+';
                s += std::to_string(u(u(5) == 0 ? 1200 : 400));
            }
        } else if (kind == 4) {  // subnormal and tiny normal range
            double d;
            uint64_t b = rng() % 0x0020000000000000ull;
            std::memcpy(&d, &b, 8);
            std::snprintf(buf, sizeof buf, "%.*e", (int)u(30), d);
            s = buf;
        } else if (kind == 5) {  // near DBL_MAX
            double d;
            uint64_t b = 0x7FEFFFFFFFFFFFFFull - (rng() % 1000);
            std::memcpy(&d, &b, 8);
            std::snprintf(buf, sizeof buf, "%.*e", 15 + (int)u(10), d);
            s = buf;
        } else if (kind == 6) {  // integers and exact decimals around 2^53
            const uint64_t v = (1ull << 53) - 500 + u(1000);
            s = std::to_string(v);
            if (u(2)) s += "." + std::to_string(u(1000000));
        } else {  // syntax noise around numbers
            const char* alpha = "0123456789.eE+-x ";
            const int n = 1 + (int)u(12);
            for (int k = 0; k < n; ++k) s += alpha[u(17)];
        }
        check(s);
    }
    std::printf("cases=%ld slow=%ld mismatches=%ld\n", n_cases, n_slow, n_fail);
    return n_fail ? 1 : 0;
}

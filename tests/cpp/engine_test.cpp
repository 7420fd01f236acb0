// TEST BUILD ONLY: the SQL route. The same CSV table and
// SQL statements go through the reference engine twice: engine_ref runs the
// reference dispatch with Mesh x Mesh rows filled by the CPU A17 composition
// (tests/cpp/engine_route_a17.hpp, oracle/_ref), engine_dev has run_batch
// routed to the device shim (tests/cpp/engine_route.hpp). Every rendered
// cell (format_double text, engine.cpp:113-117), notice and command tag must
// be identical, and the snapshot's device columns must be built once and
// then reused.
#include <cstdio>
#include <random>
#include <string>
#include <vector>

#include "engine_side.hpp"

namespace {

std::string num(double v) {
    char b[40];
    std::snprintf(b, sizeof b, "%.17g", v);
    return b;
}

std::string pt(double x, double y, double z) { return num(x) + " " + num(y) + " " + num(z); }

// a blob of n random triangles around c, as TIN Z text
std::string blob(std::mt19937_64& rng, const double c[3], double r, int n) {
    std::uniform_real_distribution<double> u(-r, r);
    std::string s = "TIN Z (";
    for (int i = 0; i < n; ++i) {
        double v[9];
        for (int k = 0; k < 9; ++k) v[k] = c[k % 3] + u(rng);
        if (i) s += ", ";
        s += "((" + pt(v[0], v[1], v[2]) + ", " + pt(v[3], v[4], v[5]) + ", " + pt(v[6], v[7], v[8]) + ", " +
             pt(v[0], v[1], v[2]) + "))";
    }
    return s + ")";
}

}  // namespace

int main() {
    std::mt19937_64 rng(1808);
    std::uniform_real_distribution<double> box(0.0, 100.0);
    std::string csv = "id,geom\n";
    int id = 1;
    for (int i = 0; i < 60; ++i) {  // meshes (some overlap the literal)
        const double c[3] = {box(rng), box(rng), box(rng)};
        csv += std::to_string(id++) + ",\"" + blob(rng, c, 6.0, 20 + (int)(rng() % 50)) + "\"\n";
    }
    for (int i = 0; i < 200; ++i) {  // drill segments
        const double x = box(rng), y = box(rng);
        csv += std::to_string(id++) + ",\"LINESTRING Z (" + pt(x, y, 100.0) + ", " + pt(x + 1, y - 2, box(rng) - 20) +
               ")\"\n";
    }
    for (int i = 0; i < 100; ++i)  // points
        csv += std::to_string(id++) + ",\"POINT Z (" + pt(box(rng), box(rng), box(rng)) + ")\"\n";
    for (int i = 0; i < 10; ++i)  // 3-point line strings: reference dispatch (TypeMismatch)
        csv += std::to_string(id++) + ",\"LINESTRING Z (0 0 0, 1 1 1, " + pt(box(rng), 2, 3) + ")\"\n";

    const double lc[3] = {50, 50, 50};
    const std::string lit = "ST_GeomFromText('" + blob(rng, lc, 25.0, 300) + "')";
    const std::string seg = "ST_GeomFromText('LINESTRING Z (10 10 10, 90 90 90)')";
    const std::vector<std::string> sqls = {
        "SELECT id, ST_3DDistance(geom, " + lit + ") FROM t",
        "SELECT id FROM t WHERE ST_3DIntersects(geom, " + lit + ")",
        "SELECT id, ST_3DDistance(" + lit + ", geom) AS d FROM t WHERE d < 20 LIMIT 40",
        "SELECT id, ST_3DDistance(geom, " + lit + ") AS d, ST_3DIntersects(geom, " + lit +
            ") AS h FROM t WHERE h OR d > 30",
        "SELECT id, ST_3DDistance(geom, " + seg + ") FROM t",
        "SELECT id, ST_Volume(geom) FROM t",
        "SELECT id, ST_3DDistance(geom, " + lit + ") FROM t",
        "SELECT id, ST_3DDistance(geom, ST_GeomFromText('POINT Z (50 50 50)')) FROM t",
        "SELECT id FROM t WHERE ST_3DIntersects(" + seg + ", geom)",
    };
    const SideResult ref = engine_ref(csv, sqls);
    const SideResult dev = engine_dev(csv, sqls);
    int bad = 0;
    std::size_t cells = 0;
    for (std::size_t s = 0; s < sqls.size(); ++s) {
        const SideStatement &a = ref.statements[s], &b = dev.statements[s];
        if (a.error != b.error || a.tag != b.tag || a.notices != b.notices || a.rows != b.rows ||
            a.batches != b.batches) {
            std::printf("MISMATCH statement %zu: ref tag=%s err=%s rows=%zu | dev tag=%s err=%s rows=%zu\n", s,
                        a.tag.c_str(), a.error.c_str(), a.rows.size(), b.tag.c_str(), b.error.c_str(), b.rows.size());
            for (std::size_t r = 0; r < a.rows.size() && r < b.rows.size(); ++r)
                if (a.rows[r] != b.rows[r]) {
                    std::string x, y;
                    for (const auto& c : a.rows[r]) x += c + " ";
                    for (const auto& c : b.rows[r]) y += c + " ";
                    std::printf("  row %zu: [%s] | [%s]\n", r, x.c_str(), y.c_str());
                    break;
                }
            for (const auto& n : a.notices) std::printf("  ref notice: %s\n", n.c_str());
            for (const auto& n : b.notices) std::printf("  dev notice: %s\n", n.c_str());
            ++bad;
        }
        for (const auto& row : a.rows) cells += row.size();
        std::printf("statement %zu: %s, %zu rows, notices=%zu%s\n", s, a.tag.c_str(), a.rows.size(),
                    a.notices.size(), a.error.empty() ? "" : (" error: " + a.error).c_str());
    }
    std::printf("device snapshot cache: adopted=%zu builds=%zu hits=%zu\n", dev.cache_adopted, dev.cache_builds,
                dev.cache_hits);
    if (dev.cache_adopted != 1 || dev.cache_builds != 0 || dev.cache_hits < 10) {
        std::printf("unexpected cache use\n");
        ++bad;
    }
    // the loader itself: the reference load_csv_text vs the device loader,
    // on the table above and on CSVs that must fail at a given line
    std::vector<std::string> csvs = {csv};
    const std::string good_tin = "\"TIN Z (((0 0 0, 1 0 0, 0 1 0, 0 0 0)))\"";
    csvs.push_back("id,geom\n1," + good_tin + "\n2,\"TIN Z (((0 0 0, 1 0 0, 0 1 0, 5 5 5)))\"\n3," + good_tin + "\n");
    csvs.push_back("id,geom\n1," + good_tin + "\n2,POINT Z (1 2)\n3,\"TIN Z (((0 0 0)))\"\n");
    csvs.push_back("1," + good_tin + "\n1," + good_tin + "\n");             // duplicate id
    csvs.push_back("1," + good_tin + "\nx," + good_tin + "\n");             // bad id
    csvs.push_back("1," + good_tin + "\n2,\"TIN Z (((0 0 0, 1 0 0\n");     // unterminated quote
    csvs.push_back("1,\"TIN Z (((0 0 0, 1 0 0, 0 1 nan, 0 0 0)))\"\n2\n"); // device error before a host error
    csvs.push_back("\r\n  \nid , WKT\r\n7 , \"POLYHEDRALSURFACE Z (((0 0 0, 1 0 0, 1 1 0, 0 1 0, 0 0 0)))\" \r\n"
                   "8,\"LINESTRING Z (0 0 0, 1 1 1)\"\n9,\"TIN Z (((0 0 0, 1 0 0, 0.5 1e-20 0, 0 0 0)))\"\n");
    csvs.push_back("");
    for (std::size_t k = 0; k < csvs.size(); ++k) {
        const std::string a = engine_ref_load(csvs[k]), b = engine_dev_load(csvs[k]);
        std::printf("load %zu: %.100s\n", k, a.c_str());
        if (a != b) {
            std::printf("LOAD MISMATCH %zu:\n  ref %.300s\n  dev %.300s\n", k, a.c_str(), b.c_str());
            ++bad;
        }
    }
    if (bad) return 1;
    std::printf("ENGINE OK (%zu cells identical)\n", cells);
    return 0;
}

// TEST BUILD ONLY. One side of build/engine_test: the reference SQL engine
// (store::load_csv_text -> Catalog -> sqlfe::execute_sql). Compiled twice:
// with -Dtindb=tindb_ref against the unmodified reference (oracle/_ref), and
// plainly against the reference sources whose engine.cpp routes run_batch
// to the device shim (tests/cpp/engine_route.hpp).
#include <tindb/engine.hpp>
#include <tindb/store.hpp>

#include <string>
#include <vector>

#include "engine_side.hpp"

#include <cstdint>
#include <cstring>

#ifdef ENGINE_SIDE_DEVICE
#include "tindb_b200/kernels.hpp"
#include "tindb_b200/store.hpp"
#define LOAD_CSV(name, text, col) tindb::store::b200::load_csv_text_b200(name, text, col).table
#else
#define LOAD_CSV(name, text, col) tindb::store::load_csv_text(name, text, col)
#endif

#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)

// The loaded table as text: ids, kinds and an FNV-1a hash of every
// coordinate's bits (or the load error's what()).
std::string CAT(ENGINE_SIDE, _load)(const std::string& csv) {
    try {
        const tindb::store::GeometryTable t = LOAD_CSV("t", csv, "geom");
        std::string out = "rows=" + std::to_string(t.records.size()) + ";";
        std::uint64_t h = 1469598103934665603ull;
        auto mix = [&](const void* p, std::size_t n) {
            const unsigned char* b = static_cast<const unsigned char*>(p);
            for (std::size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
        };
        for (const auto& r : t.records) {
            out += std::to_string(r.id) + ":" + std::to_string(r.geometry.index());
            if (const auto* m = std::get_if<tindb::TriangleMesh>(&r.geometry)) {
                out += "/" + std::to_string(m->triangles.size()) + "/" + std::to_string((int)m->source_kind) + "/" +
                       std::to_string((int)m->has_degenerate_faces);
                mix(m->triangles.data(), m->triangles.size() * sizeof(tindb::Triangle));
            } else if (const auto* p = std::get_if<tindb::Point3>(&r.geometry)) {
                mix(p, sizeof *p);
            } else if (const auto* s = std::get_if<tindb::LineSegment>(&r.geometry)) {
                mix(s, sizeof *s);
            } else if (const auto* l = std::get_if<tindb::LineString>(&r.geometry)) {
                mix(l->points.data(), l->points.size() * sizeof(tindb::Point3));
            }
            out += ",";
        }
        return out + "hash=" + std::to_string(h);
    } catch (const std::exception& e) {
        return std::string("ERR:") + e.what();
    }
}

SideResult ENGINE_SIDE(const std::string& csv, const std::vector<std::string>& sqls) {
    tindb::store::Catalog catalog;
#ifdef ENGINE_SIDE_DEVICE
    tindb::store::b200::register_table_b200(catalog, tindb::store::b200::load_csv_text_b200("t", csv, "geom"));
#else
    catalog.register_table(tindb::store::load_csv_text("t", csv, "geom"));
#endif
    const auto cfg = tindb::kernels::ExecutorConfig::parallel(4);
    SideResult out;
    for (const std::string& sql : sqls) {
        SideStatement st;
        try {
            const tindb::sqlfe::QueryResult r = tindb::sqlfe::execute_sql(sql, catalog, cfg);
            st.tag = r.command_tag;
            st.rows = r.rows;
            st.notices = r.notices;
            st.batches = r.stats.batches_run;
        } catch (const std::exception& e) {
            st.error = e.what();
        }
        out.statements.push_back(std::move(st));
    }
#ifdef ENGINE_SIDE_DEVICE
    out.cache_builds = tindb::kernels::b200::default_cache().builds();
    out.cache_hits = tindb::kernels::b200::default_cache().hits();
    out.cache_adopted = tindb::kernels::b200::default_cache().adopted();
#endif
    return out;
}

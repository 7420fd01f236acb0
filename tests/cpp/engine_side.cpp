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

#ifdef ENGINE_SIDE_DEVICE
#include "tindb_b200/kernels.hpp"
#endif

SideResult ENGINE_SIDE(const std::string& csv, const std::vector<std::string>& sqls) {
    tindb::store::Catalog catalog;
    catalog.register_table(tindb::store::load_csv_text("t", csv, "geom"));
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
#endif
    return out;
}

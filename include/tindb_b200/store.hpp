// tindb_b200 C++ shim, loader side: the reference's table loaders
// (store.hpp:52-71, store.cpp:71-160) with every mesh literal parsed on the
// device (tdb_table_from_wkt, csrc/wkt.cu) in one pass per file. Header-only;
// include next to the reference sources and link libtindb_b200.so.
//
// Semantics are load_csv_text / load_wkt_file's, line for line: the same
// record order and ids, the same header rule, the same errors (CsvError with
// the 1-based line, DuplicateId, StoreError) raised for the first offending
// line. Mesh records come back bit-identical to parse_wkt's (their faces
// are downloaded from the device store), so the host GeometryTable is the
// reference's; the device table is kept alongside for the snapshot cache
// (register_table_b200). POINT / LINESTRING literals are a few bytes each
// and go through the reference parse_wkt on the host.
#pragma once

#include <tindb/store.hpp>
#include <tindb/wkt.hpp>

#include <algorithm>
#include <cctype>
#include <charconv>
#include <fstream>
#include <memory>
#include <sstream>
#include <string>
#include <string_view>
#include <unordered_set>
#include <utility>
#include <vector>

#include "tindb_b200/kernels.hpp"

namespace tindb::store::b200 {

struct LoadedTable {
    GeometryTable table;
    std::shared_ptr<const kernels::b200::DeviceColumns> device;  // null when the table has no records
};

namespace detail {

inline std::string trim(const std::string& s) {
    std::size_t b = 0, e = s.size();
    while (b < e && std::isspace(static_cast<unsigned char>(s[b]))) ++b;
    while (e > b && std::isspace(static_cast<unsigned char>(s[e - 1]))) --e;
    return s.substr(b, e - b);
}

inline std::string lowered(std::string s) {
    for (char& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
    return s;
}

// 0 TIN Z, 1 POLYHEDRALSURFACE Z, -1 anything else (keyword only: the device
// parser decides everything after it)
inline int mesh_keyword(const std::string& wkt) {
    std::size_t p = 0;
    while (p < wkt.size() && std::isspace(static_cast<unsigned char>(wkt[p]))) ++p;
    std::size_t q = p;
    while (q < wkt.size() && (std::isalpha(static_cast<unsigned char>(wkt[q])) || wkt[q] == '_')) ++q;
    const std::string kw = lowered(wkt.substr(p, q - p));
    return kw == "tin" ? 0 : kw == "polyhedralsurface" ? 1 : -1;
}

// `id,WKT` with an optionally double-quoted WKT field ("" = one quote);
// false when the line is malformed (store.cpp:33-62 rules)
inline bool split_line(const std::string& line, std::string& id, std::string& wkt) {
    const std::size_t comma = line.find(',');
    if (comma == std::string::npos) return false;
    id = trim(line.substr(0, comma));
    const std::string rest = trim(line.substr(comma + 1));
    if (rest.empty() || rest[0] != '"') {
        wkt = rest;
        return true;
    }
    std::string out;
    std::size_t i = 1;
    for (;; ++i) {
        if (i >= rest.size()) return false;
        if (rest[i] != '"') {
            out += rest[i];
            continue;
        }
        if (i + 1 < rest.size() && rest[i + 1] == '"') {
            out += '"';
            ++i;
            continue;
        }
        break;
    }
    if (!trim(rest.substr(i + 1)).empty()) return false;
    wkt = std::move(out);
    return true;
}

struct PendingMesh {
    std::size_t record;  // index into the table's records
    std::size_t line;
    int kind;  // 0 TIN, 1 POLYHEDRALSURFACE
};

// Parse the pending mesh literals on the device, in one pass. Returns the
// device table (one object per pending mesh) and fills the records' meshes;
// on a rejected literal, *bad is its index (no table).
inline tdb_table parse_meshes(const std::vector<std::string>& texts, const std::vector<PendingMesh>& pending,
                              std::vector<GeometryRecord>& records, std::size_t* bad, std::string* what) {
    *bad = pending.size();
    if (pending.empty()) return nullptr;
    std::vector<std::uint64_t> off(texts.size() + 1, 0);
    for (std::size_t i = 0; i < texts.size(); ++i) off[i + 1] = off[i] + texts[i].size();
    std::string blob;
    blob.reserve(off.back());
    for (const std::string& t : texts) blob += t;
    tdb_table t = nullptr;
    std::uint64_t lit = 0, pos = 0;
    const int rc = tdb_table_from_wkt(blob.data(), off.data(), texts.size(), &t, &lit, &pos);
    if (rc == TDB_E_PARSE) {
        *bad = static_cast<std::size_t>(lit);
        *what = tdb_last_error();
        return nullptr;
    }
    kernels::b200::check(rc);
    try {
        std::uint64_t n = 0;
        kernels::b200::check(tdb_geom_info(t, &n, nullptr, nullptr, nullptr));
        std::vector<std::uint64_t> foff(pending.size() + 1);
        kernels::b200::check(tdb_geom_offsets(t, foff.data()));
        std::vector<Triangle> faces(n);
        kernels::b200::check(tdb_geom_download(t, reinterpret_cast<double*>(faces.data())));
        for (std::size_t k = 0; k < pending.size(); ++k) {
            TriangleMesh m;
            m.triangles.assign(faces.begin() + foff[k], faces.begin() + foff[k + 1]);
            m.source_kind = pending[k].kind == 0 ? MeshSource::Tin : MeshSource::PolyhedralSurface;
            m.refresh_degeneracy_flag();
            records[pending[k].record].geometry = std::move(m);
        }
    } catch (...) {
        tdb_table_free(t);
        throw;
    }
    return t;
}

inline LoadedTable finish(GeometryTable table, tdb_table meshes) {
    LoadedTable out;
    table.load_state = LoadState::Ready;
    if (!table.records.empty() || meshes)
        out.device = std::make_shared<const kernels::b200::DeviceColumns>(table.records, meshes);
    out.table = std::move(table);
    return out;
}

}  // namespace detail

// load_csv_text (store.hpp:62-64, store.cpp:71-122) with the mesh column on the device.
inline LoadedTable load_csv_text_b200(const std::string& table_name, const std::string& text,
                                      const std::string& geom_column = "geom") {
    GeometryTable table;
    table.name = table_name;
    table.geom_column = geom_column;
    table.load_state = LoadState::Loading;

    std::vector<detail::PendingMesh> pending;
    std::vector<std::string> mesh_texts;
    std::unordered_set<std::int64_t> ids;
    // the first error the host pass meets (raised unless a device-parsed
    // literal, all of which lie on earlier lines, fails)
    std::exception_ptr host_err;

    std::size_t line_no = 0, pos = 0;
    bool first_content = true;
    while (pos < text.size()) {
        std::size_t nl = text.find('\n', pos);
        const std::size_t end = nl == std::string::npos ? text.size() : nl;
        std::string line = text.substr(pos, end - pos);
        pos = nl == std::string::npos ? text.size() : nl + 1;
        ++line_no;
        if (!line.empty() && line.back() == '\r') line.pop_back();
        if (detail::trim(line).empty()) continue;
        std::string id_field, wkt;
        try {
            if (!detail::split_line(line, id_field, wkt))
                throw CsvError("malformed record (expected `id,WKT`)", line_no);
            if (first_content) {
                first_content = false;
                const std::string lid = detail::lowered(id_field), lg = detail::lowered(detail::trim(wkt));
                if (lid == "id" && (lg == "geometry" || lg == "wkt" || lg == detail::lowered(geom_column))) continue;
            }
            std::int64_t id = 0;
            const auto r = std::from_chars(id_field.data(), id_field.data() + id_field.size(), id);
            if (r.ec != std::errc() || r.ptr != id_field.data() + id_field.size())
                throw CsvError("invalid id \"" + id_field + "\"", line_no);
            if (!ids.insert(id).second) throw DuplicateId(id, line_no);
            const int kind = detail::mesh_keyword(wkt);
            if (kind >= 0) {
                pending.push_back({table.records.size(), line_no, kind});
                mesh_texts.push_back(std::move(wkt));
                table.records.push_back(GeometryRecord{id, Geometry{}});
            } else {
                try {
                    table.records.push_back(GeometryRecord{id, parse_wkt(wkt)});
                } catch (const WktParseError& ex) {
                    throw CsvError(std::string("WKT parse failure: ") + ex.what(), line_no);
                }
            }
        } catch (...) {
            host_err = std::current_exception();
            break;
        }
    }
    std::size_t bad = 0;
    std::string what;
    tdb_table meshes = detail::parse_meshes(mesh_texts, pending, table.records, &bad, &what);
    if (bad < pending.size()) throw CsvError("WKT parse failure: " + what, pending[bad].line);
    if (host_err) {
        tdb_table_free(meshes);
        std::rethrow_exception(host_err);
    }
    return detail::finish(std::move(table), meshes);
}

inline LoadedTable load_csv_b200(const std::string& table_name, const std::string& path,
                                 const std::string& geom_column = "geom") {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw StoreError("cannot open \"" + path + "\"");
    std::ostringstream buf;
    buf << in.rdbuf();
    if (in.bad()) throw StoreError("I/O failure reading \"" + path + "\"");
    return load_csv_text_b200(table_name, buf.str(), geom_column);
}

// load_wkt_file (store.hpp:66-71, store.cpp:133-160): one bare literal, id 1.
inline LoadedTable load_wkt_file_b200(const std::string& table_name, const std::string& path,
                                      const std::string& geom_column = "geom") {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw StoreError("cannot open \"" + path + "\"");
    std::ostringstream buf;
    buf << in.rdbuf();
    if (in.bad()) throw StoreError("I/O failure reading \"" + path + "\"");
    std::string text = buf.str();
    const char* ws = " \t\r\n";
    const std::size_t first = text.find_first_not_of(ws), last = text.find_last_not_of(ws);
    if (first == std::string::npos) throw StoreError("\"" + path + "\" is empty");
    text = text.substr(first, last - first + 1);
    GeometryTable table;
    table.name = table_name;
    table.geom_column = geom_column;
    const int kind = detail::mesh_keyword(text);
    tdb_table meshes = nullptr;
    if (kind >= 0) {
        std::vector<detail::PendingMesh> pending{{0, 1, kind}};
        table.records.push_back(GeometryRecord{1, Geometry{}});
        std::size_t bad = 0;
        std::string what;
        meshes = detail::parse_meshes({text}, pending, table.records, &bad, &what);
        if (bad == 0) throw StoreError("invalid WKT in \"" + path + "\": " + what);
    } else {
        try {
            table.records.push_back({1, parse_wkt(text)});
        } catch (const WktParseError& e) {
            throw StoreError("invalid WKT in \"" + path + "\": " + e.what());
        }
    }
    return detail::finish(std::move(table), meshes);
}

// Catalog::register_table (store.hpp:78) that also seeds the snapshot cache
// with the loader's device columns, so the first statement on the table
// does not upload it again. The seed is only taken when the published
// snapshot holds exactly the records loaded here.
inline TableSnapshot register_table_b200(Catalog& catalog, LoadedTable&& loaded,
                                         kernels::b200::SnapshotCache& cache = kernels::b200::default_cache()) {
    const std::string name = loaded.table.name;
    const GeometryRecord* data = loaded.table.records.data();
    const std::size_t size = loaded.table.records.size();
    catalog.register_table(std::move(loaded.table));
    TableSnapshot snap = catalog.scan(name);
    if (loaded.device && snap->records.data() == data && snap->records.size() == size)
        cache.adopt(snap, std::move(loaded.device));
    return snap;
}

}  // namespace tindb::store::b200

namespace tindb::b200 {

// parse_wkt (wkt.hpp:35, wkt.cpp:188) with mesh literals (TIN Z /
// POLYHEDRALSURFACE Z) parsed on the device; other literals (a few bytes)
// go to the reference parser. A rejected mesh literal raises the
// reference's WktParseError: same message, same byte position.
inline Geometry parse_wkt(std::string_view text) {
    const int kind = store::b200::detail::mesh_keyword(std::string(text));
    if (kind < 0) return ::tindb::parse_wkt(text);
    tdb_mesh m = nullptr;
    std::uint64_t pos = 0;
    const int rc = tdb_mesh_from_wkt(text.data(), text.size(), &m, &pos);
    if (rc == TDB_E_PARSE) {
        std::string what = tdb_last_error();  // the reference's what(): "<message> at position <pos>"
        const std::string tail = " at position " + std::to_string(pos);
        if (what.size() >= tail.size() && what.compare(what.size() - tail.size(), tail.size(), tail) == 0)
            what.resize(what.size() - tail.size());
        throw WktParseError(what, static_cast<std::size_t>(pos));
    }
    kernels::b200::check(rc);
    TriangleMesh mesh;
    try {
        std::uint64_t n = 0;
        kernels::b200::check(tdb_geom_info(m, &n, nullptr, nullptr, nullptr));
        mesh.triangles.resize(n);
        kernels::b200::check(tdb_geom_download(m, reinterpret_cast<double*>(mesh.triangles.data())));
    } catch (...) {
        tdb_mesh_free(m);
        throw;
    }
    tdb_mesh_free(m);
    mesh.source_kind = kind == 0 ? MeshSource::Tin : MeshSource::PolyhedralSurface;
    mesh.refresh_degeneracy_flag();
    return Geometry{std::move(mesh)};
}

}  // namespace tindb::b200

// TEST BUILD ONLY: force-included (-include) when build/ref_unit_tests
// compiles the reference's own unit tests (tests/test_batch.cpp,
// test_volume.cpp, test_distance.cpp, test_intersect.cpp, test_geometry.cpp,
// test_store.cpp, unmodified, from
// /root/reference). The operator entry points the device engine replaces
// are sent to the C++ shim
// (include/tindb_b200/kernels.hpp, store.hpp): run_batch (batch.hpp:49-51),
// mesh_volume (kernels.hpp:66), distance_to_mesh and intersects_mesh
// (kernels.hpp:68-90), parse_wkt (wkt.hpp:35) and the table loaders
// load_csv_text / load_csv / load_wkt_file (store.hpp:52-71). Everything else those tests call (the primitives
// segment_triangle_distance & co., closure validation, fixtures) is the
// reference's own code, unchanged.
#pragma once
#include <tindb/batch.hpp>
#include <tindb/kernels.hpp>

#include <tindb/store.hpp>
#include <tindb/wkt.hpp>

#include "tindb_b200/kernels.hpp"
#include "tindb_b200/store.hpp"

#define run_batch(...) ::tindb::kernels::b200::run_batch_b200(__VA_ARGS__)
#define mesh_volume(...) ::tindb::kernels::b200::mesh_volume(__VA_ARGS__)
#define distance_to_mesh(...) ::tindb::kernels::b200::distance_to_mesh(__VA_ARGS__)
#define intersects_mesh(...) ::tindb::kernels::b200::intersects_mesh(__VA_ARGS__)
#define parse_wkt(...) ::tindb::b200::parse_wkt(__VA_ARGS__)
#define load_csv_text(...) ::tindb::store::b200::load_csv_text_b200(__VA_ARGS__).table
#define load_csv(...) ::tindb::store::b200::load_csv_b200(__VA_ARGS__).table
#define load_wkt_file(...) ::tindb::store::b200::load_wkt_file_b200(__VA_ARGS__).table

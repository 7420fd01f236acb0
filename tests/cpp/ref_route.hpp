// TEST BUILD ONLY: force-included (-include) when build/ref_unit_tests
// compiles the reference's own unit tests (tests/test_batch.cpp,
// test_volume.cpp, test_distance.cpp, test_intersect.cpp, unmodified, from
// /root/reference). The operator entry points the device engine replaces
// are sent to the C++ shim
// (include/tindb_b200/kernels.hpp): run_batch (batch.hpp:49-51),
// mesh_volume (kernels.hpp:66), distance_to_mesh and intersects_mesh
// (kernels.hpp:68-90). Everything else those tests call (the primitives
// segment_triangle_distance & co., closure validation, fixtures) is the
// reference's own code, unchanged.
#pragma once
#include <tindb/batch.hpp>
#include <tindb/kernels.hpp>

#include "tindb_b200/kernels.hpp"

#define run_batch(...) ::tindb::kernels::b200::run_batch_b200(__VA_ARGS__)
#define mesh_volume(...) ::tindb::kernels::b200::mesh_volume(__VA_ARGS__)
#define distance_to_mesh(...) ::tindb::kernels::b200::distance_to_mesh(__VA_ARGS__)
#define intersects_mesh(...) ::tindb::kernels::b200::intersects_mesh(__VA_ARGS__)

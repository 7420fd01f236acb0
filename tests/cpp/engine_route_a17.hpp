// TEST BUILD ONLY (the checker side): force-included when build/engine_test
// compiles the reference engine.cpp in namespace tindb_ref. The reference
// has no Mesh x Mesh operator (batch.cpp:49,62 return TypeMismatch); the
// oracle's definition (oracle/ref_composition.cpp) is
// filled in for those rows on the CPU, so this engine is "the reference
// plus the A17 composition" — what the device route must reproduce.
#pragma once
#include <tindb/batch.hpp>
#include <tindb/kernels.hpp>

#include <cstdint>

extern "C" int ref_mesh_mesh_distance(const double* a9, std::uint64_t n, const double* b9, std::uint64_t m,
                                      std::uint64_t row_begin, std::uint64_t row_end, std::uint64_t row_stride,
                                      int threads, double* out7, std::uint64_t* pair_out);
extern "C" int ref_mesh_mesh_intersects(const double* a9, std::uint64_t n, const double* b9, std::uint64_t m,
                                        std::uint64_t row_begin, std::uint64_t row_end, std::uint64_t row_stride,
                                        int threads, std::uint64_t* pair_out);

namespace tindb::kernels {

inline std::vector<KernelResult> a17_run_batch(BatchOp op, const std::vector<store::GeometryRecord>& records,
                                               const std::optional<Geometry>& arg, const ExecutorConfig& cfg) {
    std::vector<KernelResult> out = run_batch(op, records, arg, cfg);
    if (!arg || kind_of(*arg) != GeometryKind::Mesh || (op != BatchOp::Distance && op != BatchOp::Intersects))
        return out;
    const auto& b = std::get<TriangleMesh>(*arg);
    const double* b9 = reinterpret_cast<const double*>(b.triangles.data());
    for (std::size_t i = 0; i < records.size(); ++i) {
        if (kind_of(records[i].geometry) != GeometryKind::Mesh) continue;
        const auto& a = std::get<TriangleMesh>(records[i].geometry);
        const double* a9 = reinterpret_cast<const double*>(a.triangles.data());
        const std::uint64_t n = a.triangles.size(), m = b.triangles.size();
        std::uint64_t pair = 0;
        if (op == BatchOp::Distance) {
            double o7[7];
            ref_mesh_mesh_distance(a9, n, b9, m, 0, n, 1, 4, o7, &pair);
            out[i].value = o7[0];
        } else {
            out[i].value = ref_mesh_mesh_intersects(a9, n, b9, m, 0, n, 1, 4, &pair) != 0;
        }
    }
    return out;
}

}  // namespace tindb::kernels

#define run_batch(op, records, argument, cfg) a17_run_batch(op, records, argument, cfg)

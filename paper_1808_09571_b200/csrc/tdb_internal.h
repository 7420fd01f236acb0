// Internal layout shared by the host runtime and the sm_100a kernels.
#pragma once

#include <cstdint>

namespace tdb {

// ---- device geometry store: per-face SoA planes -------------------------
// Each plane holds one double per face, n_pad entries (n_pad % 64 == 0,
// plane base 256-byte aligned => every TMA bulk copy of an even face range is
// 16-byte aligned). Planes 0..8 are the caller's coordinates, bit-for-bit
// (the exact pass reads them); the rest are per-face terms hoisted out of the
// pair loop ("per-triangle and per-edge terms hoisted").
enum Field : int {
    F_V = 0,     // V0x V0y V0z V1x V1y V1z V2x V2y V2z
    F_E = 9,     // E_j = V_{j+1} - V_j (cyclic), 3 x xyz
    F_L = 18,    // |E_j|^2
    F_IL = 21,   // 1 / |E_j|^2
    F_N = 24,    // unit normal of (V1-V0) x (V2-V0)
    F_C = 27,    // plane offset n.V0
    F_U = 28,    // dual basis: u(P) = U.(P - V0)
    F_W = 31,    //             v(P) = W.(P - V0)
    F_DEG = 34,  // 1.0 when degenerate (geometry.hpp:75, evaluated exactly)
    F_LO = 35,   // face AABB lo xyz
    F_HI = 38,   // face AABB hi xyz
    F_K = 41,    // intersects noise coefficient kappa_T = 8e-15 * |e0||e1|/|N| (+inf when N = 0)
    NF = 42
};
constexpr int kFilterPlanes = F_DEG + 1;  // planes the distance filters stage (V .. DEG)

// A-side work tile: up to kTile consecutive faces of one object.
struct Tile {
    uint64_t row0;      // first face (global index in the A store)
    uint64_t obj_row0;  // first face of the tile's object
    uint32_t count;     // faces in the tile (<= kTile)
    uint32_t obj;       // object index in the A store
};

constexpr int kTile = 128;          // A faces per CTA (one per thread)
constexpr uint64_t kChunk = 8192;   // B faces per work item
#ifndef TDB_KSB
#define TDB_KSB 32
#endif
constexpr int kSB = TDB_KSB;        // B faces per TMA-staged sub-tile
constexpr int kPlanePad = 64;

// ---- B feature blocks (the distance filter's B side) -------
// B's faces in blocks of kFB consecutive faces. Per block (fixed capacity
// kFBCap doubles), four AoS lists packed back to back from the block's base:
//   face planes   (non-degenerate faces): kFP doubles = N, U, W, 0
//   face vertices (the same faces):       kFV doubles = V (9), face index (u64 bits)
//   vertices (distinct within the block, bitwise): kVR doubles = x y z 0
//   edges    (distinct within the block, unordered vertex pair): kER doubles
//            = start P (3), E = V_k+1 - V_k (3), |E|^2, 1/|E|^2 of the first
//            face that has it
// so each kernel stages one contiguous range: [planes | vertices of faces]
// (vertex_kernel), [vertices of faces | distinct vertices] (filter_kernel),
// [edges] (edge_kernel). A pair's filter value is the minimum over its 6
// vertex/face and 9 edge/edge candidates; a shared vertex or edge is the
// same candidate for every face of the block that has it, so the filter
// evaluates it once per block.
#ifndef TDB_KFB
#define TDB_KFB 64
#endif
constexpr int kFB = TDB_KFB;
enum : int { FP_N = 0, FP_U = 3, FP_W = 6, kFP = 10 };
enum : int { FV_V = 0, FV_IDX = 9, kFV = 10 };
enum : int { ER_P = 0, ER_E = 3, ER_L = 6, ER_IL = 7, kER = 8 };
constexpr int kVR = 4;
constexpr int kFBCap = kFB * (kFP + kFV + 3 * kVR + 3 * kER);  // doubles per block (28,672 B)

// ---- A side of the shared candidates ----------------------
// Edges: per super-tile (kSuperTile consecutive tiles of one object), its
// distinct edges (unordered pair of bitwise-distinct vertices, non-degenerate
// faces only), ordered by super-tile (csrc/atiles.cu); entry = kAER doubles =
// start Q (3), E (3), |E|^2, 1/|E|^2, the two tiles that have it (u32 | u32
// << 32, equal when one), 0. The edge kernel runs kEdgeAPT x kTile
// consecutive entries per CTA.
enum : int { AR_Q = 0, AR_E = 3, AR_L = 6, AR_IL = 7, AR_TILE = 8, kAER = 10 };
#ifndef TDB_SUPERTILE
#define TDB_SUPERTILE 256
#endif
constexpr uint64_t kSuperTile = TDB_SUPERTILE;
// B side of the edge/edge candidates when the chunk allows (FULL mode, chunk
// % kBSuper == 0, i.e. full 8,192-face chunks): B's distinct edges per kBSuper
// consecutive faces (the same builder, csrc/atiles.cu), streamed by
// edge_kernel kEdgePiece entries per TMA stage.
#ifndef TDB_BSUPER
#define TDB_BSUPER 8192
#endif
constexpr uint64_t kBSuper = TDB_BSUPER;
constexpr int kEdgePiece = 256;
// Those B entries as FP32 records of kBER floats (two float4): P - o (3), E
// (3), |E|^2, 1/|E|^2, o = B's box centre; the FP32 edge/edge candidate
// (fast_pair.cuh edge_pair32, eta_f32).
constexpr int kBER = 8;
// Vertices: likewise per super-tile, kAVR doubles = x y z, two tiles (u32 |
// u32 << 32).
constexpr int kAVR = 4;

// per-object statistics (doubles): aabb lo xyz, hi xyz, max edge, max |coord|,
// max kappa (F_K) over its non-degenerate faces
constexpr int kObjStats = 9;

// Pair-filter tolerance (DESIGN.md 4.2 states and proves the bound):
//   eta(m) = kBandEdge * sqrt(L (m + 4L)) + kappa_max (m + 4L) + kBandAbs * max |coord|
// with L the max edge of the two objects, kappa_max their max F_K, m the band's
// base distance. For every pair, d~ <= d_true + eta(m) whenever d_true <= the
// band: the first term is the edge/edge solve's cancellation floor after the
// Newton-refined first parameter (<= 5.2e-8 sqrt(L (|w| + L))), the second the
// misclassification of a vertex projection / piercing on a face of
// conditioning K (<= 6.7e-16 K |w|), the third the rounding of the values.
//   band  = m (1 + kBandRel) + 2 eta(m), m = sqrt(min d~^2)   (candidates: d~ <= band)
//   done when the exact minimum D <= band - eta(m), else m = D and repeat
// kBandRel covers the 2^-20 high-word truncation of d~^2 (fast_pair.cuh).
constexpr double kBandRel = 4e-6;
constexpr double kBandEdge = 2e-7;  // 4x the proven 5.2e-8
constexpr double kBandAbs = 1e-12;

// Intersects culls ("when can the reference report a hit").
// D = diag of a box holding both triangles (or segment and triangle),
// kappa_T = F_K of triangle T (8e-15 K_T, K_T = |e0||e1|/|N| its conditioning),
// abs = kCullAbs * max |coord|:
//   one-way : all vertices of T2 beyond (kCullOne + kappa_T1) D + abs on one
//             side of T1's plane  => no directed edge of either triangle hits
//   two-way : T2 beyond (kCullTwo + kappa_T1) D + abs of T1's plane AND
//             T1 beyond (kCullTwo + kappa_T2) D + abs of T2's plane
//   apart   : the boxes of the two triangles (segment) separated by
//             kApart D + abs along an axis
// The margins cover the reference's own rounding noise (its Cramer solve at
// its 1e-12 validity edge moves the solution by <= 7.2e-3 D), not only ours.
constexpr double kCullOne = 2.5e-2;
constexpr double kCullTwo = 1.01e-12;
constexpr double kApart = 5e-2;
constexpr double kCullAbs = 1e-13;
// hit_kernel's B sub-tile (and its bounding sphere: csrc/store.cu
// geom_hit_spheres); a row whose one-way margin clears the whole sphere skips
// the sub-tile (every face of it would be culled one-way).
constexpr int kHitGroup = 128;

}  // namespace tdb

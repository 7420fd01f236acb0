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
    NF = 41
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

// per-object statistics (doubles): aabb lo xyz, hi xyz, max edge, max |coord|
constexpr int kObjStats = 8;

// Pair-filter tolerances:
//   eta   = kBandEdge * max edge + kBandAbs * max |coord|   (>= filter error
//           |d~ - d_true| plus the rounding of the reference's witnesses)
//   band  = sqrt(min d~^2) * (1 + kBandRel) + 2 eta          (candidates: d~ <= band)
//   done when the exact minimum D <= band - eta, else band = D (1 + kBandRel) + 2 eta
// kBandRel covers the 2^-20 high-word truncation of d~^2 (fast_pair.cuh).
// intersects plane cull margin:
//   tau   = kCullDiag * diag(AABB(A obj u B)) + kCullAbs * max |coord|
constexpr double kBandRel = 4e-6;
// kBandEdge: the filter's first parameter s0 comes from rcp.approx (about
// 2^-20 relative). Ericson's refinement (t for s0, then s for t) damps that by
// cos^2(theta), but when two edges pass within d << |E| of each other the
// distance error is first order: <= 0.38 * 1.2e-6 * |E| ~ 4.6e-7 |E| (4.0e-7
// |E| seen in tests/test_gpu_bounds.py over 2M adversarial pairs). 4e-6 keeps
// a ~9x margin; the band only widens by a few 1e-6 of an edge.
constexpr double kBandEdge = 4e-6;
constexpr double kBandAbs = 1e-12;
constexpr double kCullDiag = 1e-10;
constexpr double kCullAbs = 1e-13;

}  // namespace tdb

// Run partial layout and run-split limits shared by the assembly kernels
// (assembly.cuh) and the device planner (plan.cu).
#pragma once

namespace gmcp_b200 {

constexpr int kRunSamples = 128;  // planner splits longer runs (bounds per-warp work)
constexpr int kRunMasters = 8;    // local master vertices per run (planner splits)

// Partial layout (doubles) at pbase[r]. Every partial starts 32-byte aligned
// (sizes are multiples of 4 doubles) and every vector K8 reads lies in one
// aligned 4-double group, so K8 fetches it with one 256-bit load (its cost is
// L1 wavefronts per scattered load, not bytes):
//   [0..2] n  [3] energy
//   [4 + 4i .. 6 + 4i] slave gradient g_i                      (i < 3)
//   [16 + 12 bid ..] SS block bid = (0,0),(0,1),(0,2),(1,1),(1,2),(2,2), row-major, 9 of 12
//   [88 + 12m ..] master m: a_{m,0} (3) s_m | a_{m,1} (3) - | a_{m,2} (3) -  (m < M)
//   [88 + 12M + tri(m,l)] c_ml, dense upper triangle m <= l (0 when no sample has both)
// M travels in K8's contribution codes, so the partial carries no header.
constexpr int kSSBase = 16;
constexpr int kMBase = 88;
__host__ __device__ constexpr int m_base(int m) { return kMBase + 12 * m; }
__host__ __device__ constexpr int pair_base(int M) { return kMBase + 12 * M; }
__host__ __device__ constexpr int partial_size(int M) { return (pair_base(M) + M * (M + 1) / 2 + 3) & ~3; }
__host__ __device__ constexpr int tri_index(int m, int l, int M) { return m * M - m * (m - 1) / 2 + (l - m); }

}  // namespace gmcp_b200

// Run partial layout and run-split limits shared by the assembly kernels
// (assembly.cuh) and the device planner (plan.cu).
#pragma once

namespace gmcp_b200 {

constexpr int kRunSamples = 128;  // planner splits longer runs (bounds per-warp work)
constexpr int kRunMasters = 8;    // local master vertices per run (planner splits)

// Partial layout (doubles) at pbase[r] -- self-describing, so K8 needs no
// other per-run index:
//   [0] energy  [1..3] n  [4..12] slave gradients (i*3+k)
//   [13..66] SS blocks (0,0),(0,1),(0,2),(1,1),(1,2),(2,2), 9 each, row-major
//   [67] M   [68..70] slave vertex ids   [71 .. 71+M) local master vertex ids
//   [71 + M + 10m] s_m, [+1 + 3i + k] a_{m,i}[k]          (m < M)
//   [71 + 11M + tri(m,l)] c_ml, dense upper triangle m <= l (0 when no sample has both)
constexpr int kSSBase = 13;
constexpr int kMcnt = 67, kSlv = 68, kHdr = 71;
__host__ __device__ constexpr int m_base(int M) { return kHdr + M; }
__host__ __device__ constexpr int pair_base(int M) { return kHdr + 11 * M; }
__host__ __device__ constexpr int partial_size(int M) { return kHdr + 11 * M + M * (M + 1) / 2; }
__host__ __device__ constexpr int tri_index(int m, int l, int M) { return m * M - m * (m - 1) / 2 + (l - m); }

}  // namespace gmcp_b200

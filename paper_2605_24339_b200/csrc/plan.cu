// Contact-Hessian assembly plan, built on the device once per rebuild (the
// sample set is frozen between rebuilds). Everything K7 / K8 index by is made
// here from the device sample arrays with scans, one stable radix sort and a
// run-length encode -- the "segmented sort/reduce" assembly of SURVEY 8a A9:
//
//   1. slave-triangle segments: head flags + scan (samples are in reference
//      order, contact_sampling.hpp:438-468, so a segment is contiguous)
//   2. runs: one thread per segment splits it greedily at kRunSamples samples
//      or kRunMasters distinct master vertices (count pass, scan, emit pass)
//   3. per run: sorted local master table, packed per-sample local slots
//      (li4), the 64-bit set of master pairs that share a sample, and the
//      partial base (scan of partial_size(M))
//   4. per run: every (row, col) block contribution, code (pbase << 12 | M << 8
//      | role << 4 | b), plus per-row gradient entries; a stable radix sort by
//      (row, col) groups them with ascending run order preserved inside each
//      block (the order K8 sums in)
//   5. run-length encode -> BCSR columns, per-block contribution offsets;
//      row counts -> rowptr, row entry offsets
//
// The result is bitwise the plan the earlier host planner produced (same runs,
// same local tables, same pattern, same contribution order).
#include <algorithm>

#include "ctx.hpp"
#include "cubutil.cuh"
#include "partial_layout.cuh"

namespace gmcp_b200 {
namespace {

int grid_for(int64_t n, int threads) {
  const int64_t b = (n + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 64));
}

#define GRID_LOOP(i, n) \
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

__device__ __forceinline__ bool same_tri(const int32_t* sl, int64_t i, int64_t j) {
  return sl[3 * i] == sl[3 * j] && sl[3 * i + 1] == sl[3 * j + 1] && sl[3 * i + 2] == sl[3 * j + 2];
}

// 1. head[i] = 1 where a new slave triangle starts
__global__ void k_seg_heads(int64_t n, const int32_t* __restrict__ sl, int32_t* __restrict__ head) {
  GRID_LOOP(i, n) head[i] = (i == 0 || !same_tri(sl, i, i - 1)) ? 1 : 0;
}
__global__ void k_seg_starts(int64_t n, const int32_t* __restrict__ head, const int32_t* __restrict__ hscan,
                             int64_t* __restrict__ seg_start) {
  GRID_LOOP(i, n) if (head[i]) seg_start[hscan[i]] = i;
}

// 2. greedy run split of one segment (mirrors the order of the checks: a new
// run opens at the segment start, after kRunSamples samples, or when the
// sample's new master vertices would exceed kRunMasters)
template <bool Emit>
__global__ void k_runs(int64_t n_seg, const int64_t* __restrict__ seg_start, int64_t n,
                       const int32_t* __restrict__ ms, const int32_t* __restrict__ sl, int32_t* __restrict__ run_cnt,
                       const int32_t* __restrict__ run_first, int64_t* __restrict__ run_off,
                       int32_t* __restrict__ run_M, int32_t* __restrict__ run_slave) {
  GRID_LOOP(sg, n_seg) {
    const int64_t i0 = seg_start[sg], i1 = sg + 1 < n_seg ? seg_start[sg + 1] : n;
    int32_t set[kRunMasters];
    int m = 0, cnt = 0;
    int64_t start = i0;
    int r = Emit ? run_first[sg] : 0;
    auto close = [&](int64_t end) {
      (void)end;
      if (Emit) {
        run_off[r] = start;
        run_M[r] = m;
        run_slave[3 * r] = sl[3 * start];
        run_slave[3 * r + 1] = sl[3 * start + 1];
        run_slave[3 * r + 2] = sl[3 * start + 2];
        ++r;
      }
      ++cnt;
    };
    for (int64_t i = i0; i < i1; ++i) {
      int add = 0;
      for (int j = 0; j < 3; ++j) {
        const int32_t v = ms[3 * i + j];
        if (v < 0) continue;
        bool found = false;
        for (int q = 0; q < m; ++q) found |= set[q] == v;
        add += !found;
      }
      if (i > i0 && (i - start >= kRunSamples || m + add > kRunMasters)) {
        close(i);
        start = i;
        m = 0;
      }
      for (int j = 0; j < 3; ++j) {
        const int32_t v = ms[3 * i + j];
        if (v < 0) continue;
        bool found = false;
        for (int q = 0; q < m; ++q) found |= set[q] == v;
        if (!found) set[m++] = v;
      }
    }
    close(i1);
    if (!Emit) run_cnt[sg] = cnt;
  }
}

// 3. local tables per run
__global__ void k_run_sizes(int64_t R, const int32_t* __restrict__ run_M, int64_t* __restrict__ psize) {
  GRID_LOOP(r, R) psize[r] = partial_size(run_M[r]);
}

__device__ __forceinline__ int n_master_of(int8_t t) { return t == GMCP_FACE ? 3 : (t == GMCP_EDGE ? 2 : 1); }

__global__ void k_run_tables(int64_t R, const int64_t* __restrict__ run_off, const int32_t* __restrict__ lm_off,
                             const int32_t* __restrict__ ms, const int8_t* __restrict__ ty,
                             int32_t* __restrict__ lm_ids, uint32_t* __restrict__ li4,
                             unsigned long long* __restrict__ pmask, int64_t* __restrict__ ccount,
                             int64_t* __restrict__ ecount) {
  GRID_LOOP(r, R) {
    const int64_t i0 = run_off[r], i1 = run_off[r + 1];
    int32_t loc[kRunMasters];
    int M = 0;
    for (int64_t i = i0; i < i1; ++i)
      for (int j = 0; j < 3; ++j) {
        const int32_t v = ms[3 * i + j];
        if (v < 0) continue;
        bool found = false;
        for (int q = 0; q < M; ++q) found |= loc[q] == v;
        if (!found) loc[M++] = v;
      }
    for (int a = 1; a < M; ++a) {  // ascending
      const int32_t v = loc[a];
      int b = a - 1;
      while (b >= 0 && loc[b] > v) {
        loc[b + 1] = loc[b];
        --b;
      }
      loc[b + 1] = v;
    }
    for (int q = 0; q < M; ++q) lm_ids[lm_off[r] + q] = loc[q];
    unsigned long long mask = 0;
    for (int64_t i = i0; i < i1; ++i) {
      const int nm = n_master_of(ty[i]);
      int li[3] = {0, 0, 0};
      uint32_t packed = 0xffffffffu;
      for (int j = 0; j < nm; ++j) {
        const int32_t v = ms[3 * i + j];
        int lo = 0;
        while (lo < M && loc[lo] < v) ++lo;  // lower_bound
        li[j] = lo;
        packed = (packed & ~(0xffu << (8 * j))) | ((uint32_t)lo << (8 * j));
      }
      li4[i] = packed;
      for (int a = 0; a < nm; ++a)
        for (int b = 0; b < nm; ++b)
          if (li[a] <= li[b]) mask |= 1ull << (li[a] * kRunMasters + li[b]);
    }
    pmask[r] = mask;
    int diag = 0;
    for (int a = 0; a < M; ++a) diag += (int)((mask >> (a * kRunMasters + a)) & 1ull);
    const int np = __popcll(mask);
    ccount[r] = 3 * (3 + M) + 3 * M + (2 * np - diag);
    ecount[r] = 3 + M;
  }
}

// 4. contributions and row entries of one run
__global__ void k_emit(int64_t R, const int32_t* __restrict__ run_slave, const int32_t* __restrict__ lm_off,
                       const int32_t* __restrict__ lm_ids, const int64_t* __restrict__ pbase,
                       const unsigned long long* __restrict__ pmask, const int64_t* __restrict__ coff,
                       const int64_t* __restrict__ eoff, unsigned long long* __restrict__ ckey,
                       int64_t* __restrict__ cval, unsigned long long* __restrict__ ekey,
                       int64_t* __restrict__ eval) {
  GRID_LOOP(r, R) {
    const int32_t* s = run_slave + 3 * r;
    const int32_t* L = lm_ids + lm_off[r];
    const int M = lm_off[r + 1] - lm_off[r];
    const int64_t head = (pbase[r] << 12) | ((int64_t)M << 8);
    int64_t c = coff[r], e = eoff[r];
    auto key = [](int32_t row, int32_t col) {
      return ((unsigned long long)(uint32_t)row << 32) | (unsigned long long)(uint32_t)col;
    };
    for (int i = 0; i < 3; ++i) {
      ekey[e] = (unsigned long long)(uint32_t)s[i];
      eval[e++] = head | i;
      for (int b = 0; b < 3 + M; ++b) {
        ckey[c] = key(s[i], b < 3 ? s[b] : L[b - 3]);
        cval[c++] = head | (i << 4) | b;
      }
    }
    for (int k = 0; k < M; ++k) {
      ekey[e] = (unsigned long long)(uint32_t)L[k];
      eval[e++] = head | (3 + k);
      for (int b = 0; b < 3; ++b) {
        ckey[c] = key(L[k], s[b]);
        cval[c++] = head | ((3 + k) << 4) | b;
      }
    }
    const unsigned long long mask = pmask[r];
    for (int a = 0; a < M; ++a)
      for (int b = a; b < M; ++b)
        if ((mask >> (a * kRunMasters + b)) & 1ull) {
          ckey[c] = key(L[a], L[b]);
          cval[c++] = head | ((3 + a) << 4) | (3 + b);
          if (a != b) {
            ckey[c] = key(L[b], L[a]);
            cval[c++] = head | ((3 + b) << 4) | (3 + a);
          }
        }
  }
}

// 5. pattern from the sorted unique (row, col) keys
__global__ void k_block_cols(int64_t nnzb, const unsigned long long* __restrict__ uk, int32_t* __restrict__ cols,
                             int32_t* __restrict__ rowcnt) {
  GRID_LOOP(k, nnzb) {
    cols[k] = (int32_t)(uk[k] & 0xffffffffull);
    atomicAdd(&rowcnt[(int64_t)(uk[k] >> 32)], 1);  // integer counts: order-free
  }
}
__global__ void k_key_rows(int64_t n, const unsigned long long* __restrict__ keys, int32_t* __restrict__ rowcnt) {
  GRID_LOOP(k, n) atomicAdd(&rowcnt[(int64_t)keys[k]], 1);
}

template <class T>
T last_value(const DBuf<T>& b, int64_t idx, cudaStream_t s) {
  T v{};
  GMCP_CUDA(cudaMemcpyAsync(&v, b.p + idx, sizeof(T), cudaMemcpyDeviceToHost, s));
  GMCP_CUDA(cudaStreamSynchronize(s));
  return v;
}

}  // namespace

void build_assembly_plan(Ctx& c) {
  const NvtxRange nvtx_("gmcp:assembly plan");
  AssemblyPlan& P = c.plan;
  AssemblyPlan::Tmp& T = P.tmp;
  cudaStream_t s = c.stream;
  const int64_t n = c.ns;
  const int64_t N = c.n_vertices();
  P.n_rows = (int32_t)N;
  if (N >= (int64_t)INT32_MAX) throw StatusError(GMCP_ERR_CONFIG, "assembly plan: too many vertices");

  // 1. segments
  int64_t n_seg = 0;
  if (n > 0) {
    T.head.resize(n);
    T.hscan.resize(n + 1);
    k_seg_heads<<<grid_for(n, 256), 256, 0, s>>>(n, c.s_slave.p, T.head.p);
    exclusive_scan(T.head.p, T.hscan.p, n, s);
    n_seg = (int64_t)last_value(T.hscan, n - 1, s) + last_value(T.head, n - 1, s);
    T.seg_start.resize(n_seg);
    k_seg_starts<<<grid_for(n, 256), 256, 0, s>>>(n, T.head.p, T.hscan.p, T.seg_start.p);
    c.launches += 2;
  }
  // 2. runs
  int64_t R = 0;
  if (n_seg > 0) {
    T.run_cnt.resize(n_seg + 1);
    T.run_first.resize(n_seg + 1);
    k_runs<false><<<grid_for(n_seg, 128), 128, 0, s>>>(n_seg, T.seg_start.p, n, c.s_master.p, c.s_slave.p,
                                                       T.run_cnt.p, nullptr, nullptr, nullptr, nullptr);
    GMCP_CUDA(cudaMemsetAsync(T.run_cnt.p + n_seg, 0, sizeof(int32_t), s));
    exclusive_scan(T.run_cnt.p, T.run_first.p, n_seg + 1, s);
    R = last_value(T.run_first, n_seg, s);
  }
  P.n_runs = R;
  P.run_off.resize(R + 1);
  P.run_slave.resize(std::max<int64_t>(3 * R, 1));
  T.run_M.resize(R + 1);
  P.lm_off.resize(R + 1);
  P.pbase.resize(std::max<int64_t>(R, 1));
  T.psize.resize(R + 1);
  if (R > 0) {
    k_runs<true><<<grid_for(n_seg, 128), 128, 0, s>>>(n_seg, T.seg_start.p, n, c.s_master.p, c.s_slave.p, nullptr,
                                                      T.run_first.p, P.run_off.p, T.run_M.p, P.run_slave.p);
    GMCP_CUDA(cudaMemcpyAsync(P.run_off.p + R, &n, sizeof(int64_t), cudaMemcpyHostToDevice, s));
    c.launches += 2;
  }
  GMCP_CUDA(cudaMemsetAsync(T.run_M.p + R, 0, sizeof(int32_t), s));
  // 3. local tables, partial bases
  exclusive_scan(T.run_M.p, P.lm_off.p, R + 1, s);
  const int64_t n_lm = R > 0 ? (int64_t)last_value(P.lm_off, R, s) : 0;
  k_run_sizes<<<grid_for(R + 1, 256), 256, 0, s>>>(R, T.run_M.p, T.psize.p);
  GMCP_CUDA(cudaMemsetAsync(T.psize.p + R, 0, sizeof(int64_t), s));
  T.coff.resize(R + 1);  // temp: scan of psize -> pbase (+ total)
  exclusive_scan(T.psize.p, T.coff.p, R + 1, s);
  const int64_t plen = R > 0 ? last_value(T.coff, R, s) : 0;
  if (R > 0) GMCP_CUDA(cudaMemcpyAsync(P.pbase.p, T.coff.p, R * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  P.lm_ids.resize(std::max<int64_t>(n_lm, 1));
  P.li4.resize(std::max<int64_t>(n, 1));
  T.pmask.resize(std::max<int64_t>(R, 1));
  T.ccount.resize(R + 1);
  T.ecount.resize(R + 1);
  GMCP_CUDA(cudaMemsetAsync(T.ccount.p + R, 0, sizeof(int64_t), s));
  GMCP_CUDA(cudaMemsetAsync(T.ecount.p + R, 0, sizeof(int64_t), s));
  if (R > 0) {
    k_run_tables<<<grid_for(R, 128), 128, 0, s>>>(R, P.run_off.p, P.lm_off.p, c.s_master.p, c.s_type.p, P.lm_ids.p,
                                                   P.li4.p, T.pmask.p, T.ccount.p, T.ecount.p);
    ++c.launches;
  }
  c.launches += 1;
  P.partial_len = plen;
  P.partial.resize(std::max<int64_t>(plen, 1));
  // 4. contributions + entries, stable sort by (row, col) / row
  T.coff.resize(R + 1);
  T.eoff.resize(R + 1);
  exclusive_scan(T.ccount.p, T.coff.p, R + 1, s);
  exclusive_scan(T.ecount.p, T.eoff.p, R + 1, s);
  const int64_t nc = R > 0 ? last_value(T.coff, R, s) : 0;
  const int64_t ne = R > 0 ? last_value(T.eoff, R, s) : 0;
  if (nc >= (int64_t)INT32_MAX) throw StatusError(GMCP_ERR_CONFIG, "contact Hessian too large");
  for (auto* b : {&T.ckey, &T.ckey2, &T.ukey}) b->resize(std::max<int64_t>(nc, 1));
  for (auto* b : {&T.cval, &T.cval2}) b->resize(std::max<int64_t>(nc, 1));
  for (auto* b : {&T.ekey, &T.ekey2}) b->resize(std::max<int64_t>(ne, 1));
  for (auto* b : {&T.eval, &T.eval2}) b->resize(std::max<int64_t>(ne, 1));
  int rb = 1;
  while ((1ll << rb) < N) ++rb;  // row bits
  if (R > 0) {
    k_emit<<<grid_for(R, 128), 128, 0, s>>>(R, P.run_slave.p, P.lm_off.p, P.lm_ids.p, P.pbase.p, T.pmask.p, T.coff.p,
                                            T.eoff.p, T.ckey.p, T.cval.p, T.ekey.p, T.eval.p);
    ++c.launches;
    sort_pairs(T.ckey.p, T.ckey2.p, T.cval.p, T.cval2.p, nc, s, 32 + rb);
    sort_pairs(T.ekey.p, T.ekey2.p, T.eval.p, T.eval2.p, ne, s, rb);
  }
  // 5. pattern
  T.ucnt.resize(std::max<int64_t>(nc, 1));
  T.nuniq.resize(1);
  GMCP_CUDA(cudaMemsetAsync(T.nuniq.p, 0, sizeof(int32_t), s));
  if (nc > 0) run_length_encode(T.ckey2.p, T.ukey.p, T.ucnt.p, T.nuniq.p, nc, s);
  const int64_t nnzb = last_value(T.nuniq, 0, s);
  P.nnzb = nnzb;
  P.cols.resize(std::max<int64_t>(nnzb, 1));
  P.blk_off.resize(nnzb + 1);
  P.rowptr.resize(N + 1);
  P.row_ent_off.resize(N + 1);
  T.rowcnt.resize(N + 1);
  T.rowcnt.zero(s);
  if (nnzb > 0) {
    GMCP_CUDA(cudaMemsetAsync(T.ucnt.p + nnzb, 0, sizeof(int32_t), s));
    exclusive_scan(T.ucnt.p, P.blk_off.p, nnzb + 1, s);
    k_block_cols<<<grid_for(nnzb, 256), 256, 0, s>>>(nnzb, T.ukey.p, P.cols.p, T.rowcnt.p);
    ++c.launches;
  } else {
    P.blk_off.zero(s);
  }
  exclusive_scan(T.rowcnt.p, P.rowptr.p, N + 1, s);
  T.rowcnt.zero(s);
  if (ne > 0) {
    k_key_rows<<<grid_for(ne, 256), 256, 0, s>>>(ne, T.ekey2.p, T.rowcnt.p);
    ++c.launches;
  }
  exclusive_scan(T.rowcnt.p, P.row_ent_off.p, N + 1, s);
  P.contrib.resize(std::max<int64_t>(nc, 1));
  P.row_ent.resize(std::max<int64_t>(ne, 1));
  if (nc > 0) GMCP_CUDA(cudaMemcpyAsync(P.contrib.p, T.cval2.p, nc * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  if (ne > 0) GMCP_CUDA(cudaMemcpyAsync(P.row_ent.p, T.eval2.p, ne * sizeof(int64_t), cudaMemcpyDeviceToDevice, s));
  P.vals.resize(std::max<int64_t>(9 * nnzb, 1));
  c.sync();
  GMCP_CUDA(cudaGetLastError());
  P.valid = true;
}

}  // namespace gmcp_b200

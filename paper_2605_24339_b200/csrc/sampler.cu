// Broadphase (K1-K3) and mortar sampler (K4-K5), bit-exact with the reference.
// Compiled with -fmad=false: every floating-point operation below is a plain
// IEEE op in the reference's order, so candidate sets and samples are
// bitwise equal to build_candidate_pairs / build_contact_state.
//
//  K1 lbvh_build   Morton codes of master-triangle AABB centroids, CUB radix
//                  sort, Karras (2012) hierarchy, bottom-up AABB refit.
//  K2 lbvh_query   one WARP per slave triangle: breadth-first traversal with
//                  the inflated query box, lanes test one frontier node each,
//                  ballot compaction of hits / children in shared memory;
//                  count pass -> scan -> emit pass with a warp bitonic sort
//                  (the reference sorts, so traversal order is irrelevant).
//                  Per-thread stack traversal as the capacity fallback.
//                                                    contact_sampling.hpp:296-326
//  K3 features     per slave triangle (one warp) sorted-unique candidate edges /
//                  vertex features.                 contact_sampling.hpp:328-337
//  K4 point_owner  master vertex -> owning slave triangles (interior: all,
//                  else the first boundary one).     contact_sampling.hpp:403-436
//  K5 sample       one thread per (slave tri, feature) task in reference
//                  order: clip / quadrature / freeze; count -> scan -> emit.
//                                                    contact_sampling.hpp:97-215,438-485
#include <cub/cub.cuh>

#include <algorithm>

#include "ctx.hpp"
#include "kin.cuh"
#include "cubutil.cuh"

namespace gmcp_b200 {

namespace {

constexpr double kDblMax = 1.7976931348623157e308;

int grid_for(int64_t n, int threads) {
  const int64_t b = (n + threads - 1) / threads;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 64));
}

#define GRID_LOOP(i, n) for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n); i += (int64_t)gridDim.x * blockDim.x)

// ---------------------------------------------------------------------------
// K1: LBVH over master triangle boxes

struct Box {
  double lo[3], hi[3];
};

__device__ __forceinline__ Box tri_box(const double* __restrict__ x, const int32_t* t) {
  Box b;
  for (int k = 0; k < 3; ++k) {
    b.lo[k] = kDblMax;
    b.hi[k] = -kDblMax;
  }
  for (int i = 0; i < 3; ++i) {
    const d3 p = ld3(x, t[i]);
    const double v[3] = {p.x, p.y, p.z};
    for (int k = 0; k < 3; ++k) {
      b.lo[k] = dmin(b.lo[k], v[k]);
      b.hi[k] = dmax(b.hi[k], v[k]);
    }
  }
  return b;
}

__device__ __forceinline__ bool overlaps(const Box& a, const Box& b) {  // core.hpp:71-73
  for (int k = 0; k < 3; ++k)
    if (!(a.lo[k] <= b.hi[k]) || !(b.lo[k] <= a.hi[k])) return false;
  return true;
}

__global__ void k_master_boxes(int32_t n, const int32_t* __restrict__ tris, const double* __restrict__ x,
                               Box* __restrict__ boxes, unsigned long long* bounds) {
  unsigned long long lo[3] = {~0ull, ~0ull, ~0ull}, hi[3] = {0, 0, 0};
  GRID_LOOP(t, n) {
    const Box b = tri_box(x, tris + 3 * t);
    boxes[t] = b;
    for (int k = 0; k < 3; ++k) {
      const double c = 0.5 * (b.lo[k] + b.hi[k]);
      const unsigned long long o = ord_bits(c);
      lo[k] = o < lo[k] ? o : lo[k];
      hi[k] = o > hi[k] ? o : hi[k];
    }
  }
  for (int k = 0; k < 3; ++k) {
    for (int o = 16; o > 0; o >>= 1) {
      lo[k] = min(lo[k], __shfl_xor_sync(0xffffffffu, lo[k], o));
      hi[k] = max(hi[k], __shfl_xor_sync(0xffffffffu, hi[k], o));
    }
    if ((threadIdx.x & 31) == 0) {
      atomicMin(&bounds[k], lo[k]);
      atomicMax(&bounds[3 + k], hi[k]);
    }
  }
}

__device__ __forceinline__ unsigned int expand_bits(unsigned int v) {
  v = (v * 0x00010001u) & 0xFF0000FFu;
  v = (v * 0x00000101u) & 0x0F00F00Fu;
  v = (v * 0x00000011u) & 0xC30C30C3u;
  v = (v * 0x00000005u) & 0x49249249u;
  return v;
}

// Keys: Morton code of the AABB centroid (30 bits) above the triangle index
// (ib bits, unique keys). With batched scenes the scene id sits above both,
// so the hierarchy separates scenes before space.
__global__ void k_morton(int32_t n, const Box* __restrict__ boxes, const unsigned long long* __restrict__ bounds,
                         const int32_t* __restrict__ tris, const int32_t* __restrict__ vscene, int ib,
                         unsigned long long* __restrict__ keys, int32_t* __restrict__ idx) {
  double lo[3], ext[3];
  for (int k = 0; k < 3; ++k) {
    lo[k] = from_ord_bits(bounds[k]);
    const double h = from_ord_bits(bounds[3 + k]);
    ext[k] = h - lo[k] > 0 ? h - lo[k] : 1.0;
  }
  GRID_LOOP(t, n) {
    unsigned int q[3];
    for (int k = 0; k < 3; ++k) {
      const double c = 0.5 * (boxes[t].lo[k] + boxes[t].hi[k]);
      double u = (c - lo[k]) / ext[k];
      u = u < 0 ? 0 : (u > 1 ? 1 : u);
      q[k] = (unsigned int)(u * 1023.0);
    }
    const unsigned long long m = (expand_bits(q[0]) << 2) | (expand_bits(q[1]) << 1) | expand_bits(q[2]);
    const unsigned long long sc = vscene ? (unsigned long long)vscene[tris[3 * t]] : 0ull;
    keys[t] = (sc << (30 + ib)) | (m << ib) | (unsigned long long)t;  // unique keys: index breaks ties
    idx[t] = (int32_t)t;
  }
}

__device__ __forceinline__ int delta(const unsigned long long* k, int n, int i, int j) {
  if (j < 0 || j >= n) return -1;
  return __clzll(k[i] ^ k[j]);
}

// Karras 2012: internal nodes 0..n-2, leaves n-1..2n-2.
__global__ void k_karras(int n, const unsigned long long* __restrict__ k, int32_t* __restrict__ left,
                         int32_t* __restrict__ right, int32_t* __restrict__ parent) {
  GRID_LOOP(ii, n - 1) {
    const int i = (int)ii;
    const int d = (delta(k, n, i, i + 1) - delta(k, n, i, i - 1)) >= 0 ? 1 : -1;
    const int dmin_ = delta(k, n, i, i - d);
    int lmax = 2;
    while (delta(k, n, i, i + lmax * d) > dmin_) lmax *= 2;
    int l = 0;
    for (int t = lmax / 2; t >= 1; t /= 2)
      if (delta(k, n, i, i + (l + t) * d) > dmin_) l += t;
    const int j = i + l * d;
    const int dnode = delta(k, n, i, j);
    int s = 0;
    for (int div = 2;; div *= 2) {
      const int t = (l + div - 1) / div;
      if (delta(k, n, i, i + (s + t) * d) > dnode) s += t;
      if (t == 1) break;
    }
    const int gamma = i + s * d + min(d, 0);
    const int lo = min(i, j), hi = max(i, j);
    const int L = (lo == gamma) ? (n - 1 + gamma) : gamma;
    const int R = (hi == gamma + 1) ? (n - 1 + gamma + 1) : gamma + 1;
    left[i] = L;
    right[i] = R;
    parent[L] = i;
    parent[R] = i;
  }
}

__device__ __forceinline__ Box ldcg_box(const Box* b) {  // L2 view: written by other SMs
  Box r;
  const double* p = reinterpret_cast<const double*>(b);
  for (int k = 0; k < 3; ++k) {
    r.lo[k] = __ldcg(p + k);
    r.hi[k] = __ldcg(p + 3 + k);
  }
  return r;
}

// Bottom-up AABB refit (one thread per leaf; the second child to arrive
// merges). With batched scenes each node also records its [min, max] scene.
__global__ void k_refit(int n, const int32_t* __restrict__ sorted_idx, const Box* __restrict__ tri_boxes,
                        const int32_t* __restrict__ left, const int32_t* __restrict__ right,
                        const int32_t* __restrict__ parent, Box* nodes, int32_t* flags,
                        const int32_t* __restrict__ tris, const int32_t* __restrict__ vscene, int2* srange) {
  GRID_LOOP(t, n) {
    int node = n - 1 + (int)t;
    const int32_t tri = sorted_idx[t];
    nodes[node] = tri_boxes[tri];
    if (vscene) {
      const int sc = vscene[tris[3 * tri]];
      srange[node] = make_int2(sc, sc);
    }
    if (n == 1) continue;
    __threadfence();
    int p = parent[node];
    while (p >= 0) {
      if (atomicAdd(&flags[p], 1) == 0) break;  // first arrival: sibling not ready
      __threadfence();
      const int lc = __ldcg(left + p), rc = __ldcg(right + p);
      const Box a = ldcg_box(nodes + lc), b = ldcg_box(nodes + rc);
      Box u;
      for (int k2 = 0; k2 < 3; ++k2) {
        u.lo[k2] = dmin(a.lo[k2], b.lo[k2]);
        u.hi[k2] = dmax(a.hi[k2], b.hi[k2]);
      }
      nodes[p] = u;
      if (vscene) {
        const int* ra = reinterpret_cast<const int*>(srange + lc);
        const int* rb = reinterpret_cast<const int*>(srange + rc);
        srange[p] = make_int2(min(__ldcg(ra), __ldcg(rb)), max(__ldcg(ra + 1), __ldcg(rb + 1)));
      }
      __threadfence();
      p = p == 0 ? -1 : parent[p];
    }
  }
}

// ---------------------------------------------------------------------------
// K2: queries. mode 0 counts, mode 1 emits + sorts per slave tri.

__device__ __forceinline__ void isort(int32_t* a, int n) {
  for (int i = 1; i < n; ++i) {
    const int32_t v = a[i];
    int j = i - 1;
    while (j >= 0 && a[j] > v) {
      a[j + 1] = a[j];
      --j;
    }
    a[j + 1] = v;
  }
}
__device__ __forceinline__ int sort_unique(int32_t* a, int n) {
  isort(a, n);
  if (n == 0) return 0;
  int k = 1;
  for (int i = 1; i < n; ++i)
    if (a[i] != a[k - 1]) a[k++] = a[i];
  return k;
}

template <int Mode>
__global__ void k_query(int32_t nst, const int32_t* __restrict__ stris, const double* __restrict__ x, double r,
                        int n_leaf, const Box* __restrict__ nodes, const int32_t* __restrict__ left,
                        const int32_t* __restrict__ right, const int32_t* __restrict__ sorted_idx,
                        int64_t* __restrict__ cnt, const int64_t* __restrict__ off, int32_t* __restrict__ out,
                        int* overflow, const int32_t* __restrict__ vscene, const int2* __restrict__ srange,
                        const uint8_t* __restrict__ scene_mask) {
  GRID_LOOP(st, nst) {
    const int qs = vscene ? vscene[stris[3 * st]] : -1;  // batched scenes: own scene only
    if (scene_mask && !scene_mask[qs]) {  // scene not being re-sampled
      if (!Mode) cnt[st] = 0;
      continue;
    }
    Box q = tri_box(x, stris + 3 * st);
    for (int k = 0; k < 3; ++k) {  // Aabb::inflated, core.hpp:77-82
      q.lo[k] = q.lo[k] - r;
      q.hi[k] = q.hi[k] + r;
    }
    int stack[64];
    int top = 0;
    stack[top++] = n_leaf == 1 ? 0 : 0;
    int64_t c = 0;
    const int64_t base = Mode ? off[st] : 0;
    while (top > 0) {
      const int node = stack[--top];
      if (qs >= 0) {
        const int2 sr = srange[node];
        if (qs < sr.x || qs > sr.y) continue;
      }
      if (!overlaps(nodes[node], q)) continue;
      if (node >= n_leaf - 1) {
        if (Mode) out[base + c] = sorted_idx[node - (n_leaf - 1)];
        ++c;
      } else {
        if (top + 2 > 64) {
          atomicExch(overflow, 1);
          break;
        }
        stack[top++] = right[node];
        stack[top++] = left[node];
      }
    }
    if (Mode) isort(out + base, (int)c);
    else cnt[st] = c;
  }
}

// K2 (default): warp-cooperative traversal, one warp per slave triangle.
// The warp walks the LBVH breadth-first: each lane tests one node of the
// current frontier (scene range + Aabb::overlaps against the inflated query
// box), and ballot / popcount compaction appends the leaves hit to the warp's
// hit list and the children of the internal nodes hit to the next frontier,
// all in shared memory. The hits are then sorted by a warp bitonic sort
// (the reference sorts, contact_sampling.hpp:296-326, so the traversal order
// is irrelevant). A frontier or hit list beyond the warp's capacity raises
// *wovf and the host re-runs the per-thread kernels (k_query).
constexpr int kQW = 4;          // warps per block
constexpr int kFront = 256;     // frontier capacity per warp
constexpr int kHitCap = 512;    // hits per warp

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ascending bitonic sort of a[0, n) (n a power of two, <= kHitCap) by one warp
__device__ __forceinline__ void warp_bitonic(int32_t* a, int n) {
  const int lane = threadIdx.x & 31;
  for (int k = 2; k <= n; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < n; i += 32) {
        const int l = i ^ j;
        if (l > i) {
          const int32_t x0 = a[i], x1 = a[l];
          if ((x0 > x1) == ((i & k) == 0)) {
            a[i] = x1;
            a[l] = x0;
          }
        }
      }
      __syncwarp();
    }
}

__device__ __forceinline__ int pow2_at_least(int n) {
  int p = 32;
  while (p < n) p <<= 1;
  return p;
}

template <int Mode>
__global__ void __launch_bounds__(32 * kQW) k_query_warp(
    int32_t nst, const int32_t* __restrict__ stris, const double* __restrict__ x, double r, int n_leaf,
    const Box* __restrict__ nodes, const int32_t* __restrict__ left, const int32_t* __restrict__ right,
    const int32_t* __restrict__ sorted_idx, int64_t* __restrict__ cnt, const int64_t* __restrict__ off,
    int32_t* __restrict__ out, int* wovf, const int32_t* __restrict__ vscene, const int2* __restrict__ srange,
    const uint8_t* __restrict__ scene_mask) {
  __shared__ int32_t fr[kQW][2][kFront];
  __shared__ int32_t hits[kQW][kHitCap];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int32_t* H = hits[w];
  const unsigned lt = lanemask_lt();
  for (int64_t st = blockIdx.x * (int64_t)kQW + w; st < nst; st += (int64_t)gridDim.x * kQW) {
    const int qs = vscene ? vscene[stris[3 * st]] : -1;  // batched scenes: own scene only
    if (scene_mask && !scene_mask[qs]) {  // scene not being re-sampled
      if (!Mode && lane == 0) cnt[st] = 0;
      continue;
    }
    Box q = tri_box(x, stris + 3 * st);
    for (int k = 0; k < 3; ++k) {  // Aabb::inflated, core.hpp:77-82
      q.lo[k] = q.lo[k] - r;
      q.hi[k] = q.hi[k] + r;
    }
    int32_t* F0 = fr[w][0];
    int32_t* F1 = fr[w][1];
    if (lane == 0) F0[0] = 0;  // root (the single leaf when n_leaf == 1)
    __syncwarp();
    int nf = 1, nh = 0;
    bool ovf = false;
    while (nf > 0 && !ovf) {
      int nn = 0;
      for (int b0 = 0; b0 < nf; b0 += 32) {
        const int i = b0 + lane;
        int node = -1;
        bool hit = false, push = false;
        if (i < nf) {
          node = F0[i];
          bool ok = true;
          if (qs >= 0) {
            const int2 sr = srange[node];
            ok = !(qs < sr.x || qs > sr.y);
          }
          if (ok && overlaps(nodes[node], q)) {
            if (node >= n_leaf - 1) hit = true;
            else push = true;
          }
        }
        const unsigned hb = __ballot_sync(0xffffffffu, hit), pb = __ballot_sync(0xffffffffu, push);
        const int hpos = nh + __popc(hb & lt), ppos = nn + 2 * __popc(pb & lt);
        if (hit && hpos < kHitCap) H[hpos] = sorted_idx[node - (n_leaf - 1)];
        if (push && ppos + 1 < kFront) {
          F1[ppos] = left[node];
          F1[ppos + 1] = right[node];
        }
        nh += __popc(hb);
        nn += 2 * __popc(pb);
      }
      if (nn > kFront || nh > kHitCap) ovf = true;
      __syncwarp();
      int32_t* t = F0;
      F0 = F1;
      F1 = t;
      nf = nn;
    }
    if (ovf) {
      if (lane == 0) atomicExch(wovf, 1);
      continue;
    }
    if (!Mode) {
      if (lane == 0) cnt[st] = nh;
      continue;
    }
    const int n2 = pow2_at_least(nh);
    for (int i = nh + lane; i < n2; i += 32) H[i] = 0x7fffffff;
    __syncwarp();
    warp_bitonic(H, n2);
    const int64_t base = off[st];
    for (int i = lane; i < nh; i += 32) out[base + i] = H[i];
    __syncwarp();
  }
}

// K3 (default): the same per warp. A warp gathers its slave triangle's
// candidate edges and vertex features (lower_bound into master.verts) into
// shared memory, bitonic-sorts both lists, and keeps the first of each run of
// equal ids (ballot compaction). Over kHitCap raw ids raises *wovf.
__global__ void __launch_bounds__(32 * kQW) k_features_warp(
    int32_t nst, const int64_t* __restrict__ tri_off, const int32_t* __restrict__ tri_ids,
    const int32_t* __restrict__ mtris, const int32_t* __restrict__ mtri_edges, const int32_t* __restrict__ mverts,
    int32_t n_mverts, int32_t* __restrict__ tmp_e, int32_t* __restrict__ tmp_v, int64_t* __restrict__ ecnt,
    int64_t* __restrict__ vcnt, int* wovf) {
  __shared__ int32_t bufE[kQW][kHitCap], bufV[kQW][kHitCap];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int32_t* E = bufE[w];
  int32_t* V = bufV[w];
  const unsigned lt = lanemask_lt();
  for (int64_t st = blockIdx.x * (int64_t)kQW + w; st < nst; st += (int64_t)gridDim.x * kQW) {
    const int64_t a = tri_off[st], b = tri_off[st + 1];
    const int k = (int)(3 * (b - a));
    if (k > kHitCap) {
      if (lane == 0) atomicExch(wovf, 1);
      continue;
    }
    for (int j = lane; j < k; j += 32) {
      const int mt = tri_ids[a + j / 3], e = j % 3;
      E[j] = mtri_edges[3 * mt + e];
      const int gv = mtris[3 * mt + e];
      int lo = 0, hi = n_mverts;  // lower_bound into master.verts
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (mverts[mid] < gv) lo = mid + 1; else hi = mid;
      }
      V[j] = lo;
    }
    const int n2 = pow2_at_least(k);
    for (int j = k + lane; j < n2; j += 32) E[j] = V[j] = 0x7fffffff;
    __syncwarp();
    warp_bitonic(E, n2);
    warp_bitonic(V, n2);
    int32_t* oe = tmp_e + 3 * a;
    int32_t* ov = tmp_v + 3 * a;
    int ue = 0, uv = 0;
    for (int b0 = 0; b0 < k; b0 += 32) {
      const int j = b0 + lane;
      const bool fe = j < k && (j == 0 || E[j] != E[j - 1]);
      const bool fv = j < k && (j == 0 || V[j] != V[j - 1]);
      const unsigned be = __ballot_sync(0xffffffffu, fe), bv = __ballot_sync(0xffffffffu, fv);
      if (fe) oe[ue + __popc(be & lt)] = E[j];
      if (fv) ov[uv + __popc(bv & lt)] = V[j];
      ue += __popc(be);
      uv += __popc(bv);
    }
    if (lane == 0) {
      ecnt[st] = ue;
      vcnt[st] = uv;
    }
    __syncwarp();
  }
}

// K3: candidate edges / vertex features per slave tri (sorted unique).
// Writes into tmp at 3*tri_off[st] and the unique counts.
__global__ void k_features(int32_t nst, const int64_t* __restrict__ tri_off, const int32_t* __restrict__ tri_ids,
                           const int32_t* __restrict__ mtris, const int32_t* __restrict__ mtri_edges,
                           const int32_t* __restrict__ mverts, int32_t n_mverts, int32_t* __restrict__ tmp_e,
                           int32_t* __restrict__ tmp_v, int64_t* __restrict__ ecnt, int64_t* __restrict__ vcnt) {
  GRID_LOOP(st, nst) {
    const int64_t a = tri_off[st], b = tri_off[st + 1];
    int32_t* E = tmp_e + 3 * a;
    int32_t* V = tmp_v + 3 * a;
    int k = 0;
    for (int64_t i = a; i < b; ++i) {
      const int mt = tri_ids[i];
      for (int e = 0; e < 3; ++e) {
        E[k] = mtri_edges[3 * mt + e];
        const int gv = mtris[3 * mt + e];
        int lo = 0, hi = n_mverts;  // lower_bound into master.verts
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (mverts[mid] < gv) lo = mid + 1; else hi = mid;
        }
        V[k] = lo;
        ++k;
      }
    }
    ecnt[st] = sort_unique(E, k);
    vcnt[st] = sort_unique(V, k);
  }
}

__global__ void k_compact(int32_t nst, const int64_t* __restrict__ tri_off, const int32_t* __restrict__ tmp,
                          const int64_t* __restrict__ off, int32_t* __restrict__ out) {
  GRID_LOOP(st, nst) {
    const int32_t* src = tmp + 3 * tri_off[st];
    for (int64_t i = off[st]; i < off[st + 1]; ++i) out[i] = src[i - off[st]];
  }
}

// ---------------------------------------------------------------------------
// geometry (reference op order; this TU has no FMA contraction)

struct Frame {
  d3 origin, t1, t2, n;
};

// geometry.hpp:14-21
__device__ __forceinline__ bool triangle_normal(d3 a, d3 b, d3 c, d3& n) {
  const d3 cr = cross(b - a, c - a);
  const d3 lo = mk3(dmin(dmin(dmin(kDblMax, a.x), b.x), c.x), dmin(dmin(dmin(kDblMax, a.y), b.y), c.y),
                    dmin(dmin(dmin(kDblMax, a.z), b.z), c.z));
  const d3 hi = mk3(dmax(dmax(dmax(-kDblMax, a.x), b.x), c.x), dmax(dmax(dmax(-kDblMax, a.y), b.y), c.y),
                    dmax(dmax(dmax(-kDblMax, a.z), b.z), c.z));
  const double diag2 = norm(hi - lo);
  const double area_eps = 1e-12 * diag2 * diag2;
  if (0.5 * norm(cr) <= area_eps) return false;
  n = unit(cr);
  return true;
}
// geometry.hpp:127-134
__device__ __forceinline__ bool tangent_frame(d3 a, d3 b, d3 c, Frame& f) {
  if (!triangle_normal(a, b, c, f.n)) return false;
  f.origin = a;
  f.t1 = unit(b - a);
  f.t2 = cross(f.n, f.t1);
  return true;
}
__device__ __forceinline__ d2 to_plane(const Frame& f, d3 p) {
  const d3 d = p - f.origin;
  return d2{dot(d, f.t1), dot(d, f.t2)};
}
// geometry.hpp:101-103
__device__ __forceinline__ double signed_area_2d(d2 a, d2 b, d2 c) {
  return 0.5 * ((b.x - a.x) * (c.y - a.y) - (b.y - a.y) * (c.x - a.x));
}
// geometry.hpp:106-114
__device__ __forceinline__ bool barycentric_2d(d2 p, d2 a, d2 b, d2 c, d3& out) {
  const double area = signed_area_2d(a, b, c);
  const double diag = dmax(dmax(norm2(b - a), norm2(c - a)), norm2(c - b));
  if (fabs(area) <= 1e-14 * diag * diag) return false;
  const double u = signed_area_2d(p, b, c) / area;
  const double v = signed_area_2d(a, p, c) / area;
  out = mk3(u, v, 1.0 - u - v);
  return true;
}
__device__ __forceinline__ double hermite_step(double x, double delta) {  // barrier.hpp:69-74
  if (x <= 0) return 0;
  if (x >= delta) return 1;
  const double t = x / delta;
  return t * t * (3.0 - 2.0 * t);
}
__device__ __forceinline__ double adaptive_eps(double g, double eps_max) { return dmin(0.9 * g, eps_max); }
__device__ __forceinline__ double min3(d3 a) { return dmin(dmin(a.x, a.y), a.z); }
__device__ __forceinline__ d3 clamp_bary(d3 b) {  // contact_sampling.hpp:80-83
  b = mk3(dmax(b.x, 0.0), dmax(b.y, 0.0), dmax(b.z, 0.0));
  const double s = b.x + b.y + b.z;
  return b / s;
}
__device__ __forceinline__ double local_scale(const d3* s) {  // contact_sampling.hpp:88-90
  return (norm(s[1] - s[0]) + norm(s[2] - s[0]) + norm(s[2] - s[1])) / 3.0;
}

// quadrature.hpp:20-81
__device__ __forceinline__ int tri_quad(int order, double q[6][4]) {
  switch (order) {
    case 1:
      q[0][0] = q[0][1] = q[0][2] = 1.0 / 3.0;
      q[0][3] = 1.0;
      return 1;
    case 2: {
      const double a = 2.0 / 3.0, b = 1.0 / 6.0, w = 1.0 / 3.0;
      const double t[3][4] = {{a, b, b, w}, {b, a, b, w}, {b, b, a, w}};
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 4; ++j) q[i][j] = t[i][j];
      return 3;
    }
    case 3: {
      const double a = 0.659027622374092, b = 0.231933368553031, c = 0.109039009072877, w = 1.0 / 6.0;
      const double t[6][4] = {{a, b, c, w}, {a, c, b, w}, {b, a, c, w}, {b, c, a, w}, {c, a, b, w}, {c, b, a, w}};
      for (int i = 0; i < 6; ++i)
        for (int j = 0; j < 4; ++j) q[i][j] = t[i][j];
      return 6;
    }
    default: {
      const double a1 = 0.108103018168070, b1 = 0.445948490915965, w1 = 0.223381589678011;
      const double a2 = 0.816847572980459, b2 = 0.091576213509771, w2 = 0.109951743655322;
      const double t[6][4] = {{a1, b1, b1, w1}, {b1, a1, b1, w1}, {b1, b1, a1, w1},
                              {a2, b2, b2, w2}, {b2, a2, b2, w2}, {b2, b2, a2, w2}};
      for (int i = 0; i < 6; ++i)
        for (int j = 0; j < 4; ++j) q[i][j] = t[i][j];
      return 6;
    }
  }
}
__device__ __forceinline__ int seg_quad(int points, double q[5][2]) {
  const double x2[2] = {-0.5773502691896257, 0.5773502691896257}, w2[2] = {1.0, 1.0};
  const double x3[3] = {-0.7745966692414834, 0.0, 0.7745966692414834}, w3[3] = {5.0 / 9.0, 8.0 / 9.0, 5.0 / 9.0};
  const double x4[4] = {-0.8611363115940526, -0.3399810435848563, 0.3399810435848563, 0.8611363115940526};
  const double w4[4] = {0.3478548451374538, 0.6521451548625461, 0.6521451548625461, 0.3478548451374538};
  const double x5[5] = {-0.9061798459386640, -0.5384693101056831, 0.0, 0.5384693101056831, 0.9061798459386640};
  const double w5[5] = {0.2369268850561891, 0.4786286704993665, 0.5688888888888889, 0.4786286704993665,
                        0.2369268850561891};
  const double *xs, *ws;
  switch (points) {
    case 1:
      q[0][0] = 0.5;
      q[0][1] = 1.0;
      return 1;
    case 2: xs = x2; ws = w2; break;
    case 3: xs = x3; ws = w3; break;
    case 4: xs = x4; ws = w4; break;
    default: xs = x5; ws = w5; points = 5; break;
  }
  for (int i = 0; i < points; ++i) {
    q[i][0] = 0.5 * (1.0 + xs[i]);
    q[i][1] = 0.5 * ws[i];
  }
  return points;
}

// ---------------------------------------------------------------------------
// K4: point ownership

struct SamplerArgs {
  const double* x;
  const double* eps_ref;
  int32_t nst;
  const int32_t* stris;
  const int32_t* mtris;
  const int32_t* medges;
  const int32_t* mverts;
  gmcp_barrier_params P;
};

// One thread per master vertex feature mv: walks the ascending slave tris
// listing mv (CSR by mv) and emits the owning tris (count or write).
template <int Mode>
__global__ void k_point_owner(SamplerArgs A, int32_t nmv, const int64_t* __restrict__ by_off,
                              const int32_t* __restrict__ by_st, int64_t* __restrict__ cnt,
                              const int64_t* __restrict__ off, unsigned long long* __restrict__ keys,
                              unsigned long long* err) {
  GRID_LOOP(mv, nmv) {
    const d3 v = ld3(A.x, A.mverts[mv]);
    int first_boundary = -1;
    bool any_interior = false;
    int64_t c = 0;
    const int64_t b0 = by_off[mv], b1 = by_off[mv + 1];
    for (int pass = 0; pass < 2; ++pass) {
      if (pass == 1 && !any_interior) break;
      for (int64_t k = b0; k < b1; ++k) {
        const int st = by_st[k];
        const d3 s[3] = {ld3(A.x, A.stris[3 * st]), ld3(A.x, A.stris[3 * st + 1]), ld3(A.x, A.stris[3 * st + 2])};
        Frame f;
        d3 bary;
        if (!tangent_frame(s[0], s[1], s[2], f) ||
            !barycentric_2d(to_plane(f, v), to_plane(f, s[0]), to_plane(f, s[1]), to_plane(f, s[2]), bary)) {
          atomicMin(err, 0ull);  // ownership errors precede every emission error
          break;
        }
        const double mn = min3(bary);
        if (mn < -1e-12) continue;
        if (pass == 0) {
          if (mn > 1e-9) any_interior = true;
          else if (first_boundary < 0) first_boundary = st;
        } else if (mn > 1e-9) {
          if (Mode) keys[off[mv] + c] = ((unsigned long long)st << 32) | (unsigned int)mv;
          ++c;
        }
      }
    }
    if (!any_interior && first_boundary >= 0) {
      if (Mode) keys[off[mv] + c] = ((unsigned long long)first_boundary << 32) | (unsigned int)mv;
      ++c;
    }
    if (!Mode) cnt[mv] = c;
  }
}

// ---------------------------------------------------------------------------
// K5: sampling tasks. task = (slave tri, kind, feature), reference order.

struct Out {
  int8_t* type;
  int32_t *slave, *master;
  double *beta_s, *beta_m, *eta, *weight, *gamma, *eps, *g_ref;
  // single-pass mode (k_sample<2>): records land unordered at warp-aggregated
  // slots of a staging buffer, keyed (task << 5 | k) for the ordering sort
  uint32_t* key = nullptr;
  unsigned int* ctr = nullptr;
  int64_t cap = 0;
};

struct SampleRec {
  int8_t type;
  int32_t master[3];
  d3 bs, bm;
  double eta, weight, gamma, g;
};

// freeze (contact_sampling.hpp:471-485): returns false if the sample is dropped;
// sets g_ref/eps. err_code: 0 ok, 1 degenerate at eps_reference.
__device__ __forceinline__ bool freeze(const SamplerArgs& A, const int32_t* sid, const SampleRec& r, double& g_ref,
                                       double& eps, bool& err) {
  err = false;
  if (!(r.g > 0)) return false;  // g_now == r.g bitwise (same normal, xs, xm)
  g_ref = r.g;
  if (A.eps_ref) {
    const double* X = A.eps_ref;
    const d3 a0 = ld3(X, sid[0]), a1 = ld3(X, sid[1]), a2 = ld3(X, sid[2]);
    d3 n;
    if (!triangle_normal(a0, a1, a2, n)) {
      err = true;
      return false;
    }
    const d3 xs = (r.bs.x * a0 + r.bs.y * a1) + r.bs.z * a2;
    d3 xm;
    if (r.type == GMCP_FACE)
      xm = (r.bm.x * ld3(X, r.master[0]) + r.bm.y * ld3(X, r.master[1])) + r.bm.z * ld3(X, r.master[2]);
    else if (r.type == GMCP_EDGE)
      xm = (1.0 - r.eta) * ld3(X, r.master[0]) + r.eta * ld3(X, r.master[1]);
    else
      xm = ld3(X, r.master[0]);
    const double gs = dot(n, xm - xs);
    if (gs > 0) g_ref = gs;
  }
  eps = adaptive_eps(g_ref, A.P.eps_max);
  return true;
}

template <int Mode>
__device__ __forceinline__ void put(const SamplerArgs& A, const int32_t* sid, const SampleRec& r, int64_t& c,
                                    int64_t base, const Out& O, bool& err, int key_k = -1) {
  // key_k >= 0 (two-phase face sampling): the record's order key within its
  // task is its (sub-triangle, quadrature point) index, monotone in the
  // reference order; otherwise the running count c
  double g_ref, eps;
  if (!freeze(A, sid, r, g_ref, eps, err)) return;
  if (Mode) {
    int64_t i;
    if (Mode == 2) {  // base = task index; one atomic per group of lanes emitting together
      const unsigned am = __activemask();
      const int lane = threadIdx.x & 31, leader = __ffs(am) - 1;
      unsigned lt;
      asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
      unsigned b0 = 0;
      if (lane == leader) b0 = atomicAdd(O.ctr, (unsigned)__popc(am));
      b0 = __shfl_sync(am, b0, leader);
      i = (int64_t)b0 + __popc(am & lt);
      if (i >= O.cap) {  // staging full: counted, not stored (the host re-runs with room)
        ++c;
        return;
      }
      O.key[i] = ((uint32_t)base << 5) | (uint32_t)(key_k >= 0 ? key_k : c);
    } else {
      i = base + c;
    }
    O.type[i] = r.type;
    for (int k = 0; k < 3; ++k) {
      O.slave[3 * i + k] = sid[k];
      O.master[3 * i + k] = r.master[k];
    }
    O.beta_s[3 * i] = r.bs.x;
    O.beta_s[3 * i + 1] = r.bs.y;
    O.beta_s[3 * i + 2] = r.bs.z;
    O.beta_m[3 * i] = r.bm.x;
    O.beta_m[3 * i + 1] = r.bm.y;
    O.beta_m[3 * i + 2] = r.bm.z;
    O.eta[i] = r.eta;
    O.weight[i] = r.weight;
    O.gamma[i] = r.gamma;
    O.eps[i] = eps;
    O.g_ref[i] = g_ref;
  }
  ++c;
}

// Sutherland-Hodgman, contact_sampling.hpp:39-58
__device__ __forceinline__ int clip_polygon(d2* poly, int n, const d2* tri) {
  d2 out[12];
  for (int e = 0; e < 3; ++e) {
    if (n < 3) break;
    const d2 a = tri[e];
    const d2 dir = tri[(e + 1) % 3] - a;
    int m = 0;
    for (int i = 0; i < n; ++i) {
      const d2 p = poly[i], q = poly[(i + 1) % n];
      const double dp = cross2(dir, p - a);
      const double dq = cross2(dir, q - a);
      if (dp >= 0) out[m++] = p;
      if ((dp >= 0) != (dq >= 0)) out[m++] = p + (dp / (dp - dq)) * (q - p);
    }
    for (int i = 0; i < m; ++i) poly[i] = out[i];
    n = m;
  }
  return n;
}
__device__ __forceinline__ int merge_close(d2* poly, int n, double tol) {  // :60-66
  d2 out[12];
  int m = 0;
  for (int i = 0; i < n; ++i)
    if (m == 0 || norm2(poly[i] - out[m - 1]) > tol) out[m++] = poly[i];
  while (m >= 2 && norm2(out[0] - out[m - 1]) <= tol) --m;
  for (int i = 0; i < m; ++i) poly[i] = out[i];
  return m;
}
__device__ __forceinline__ double polygon_area(const d2* poly, int n) {  // :68-76
  double twice = 0;
  for (int i = 0; i < n; ++i) twice += cross2(poly[i], poly[(i + 1) % n]);
  return 0.5 * twice;
}

// task kinds
constexpr int kFace = 0, kEdge = 1, kPoint = 2;

template <int Mode>
__global__ void __launch_bounds__(128) k_sample(SamplerArgs A, int64_t ntask, const int32_t* __restrict__ task_st,
                                                const int32_t* __restrict__ task_feat,
                                                const int8_t* __restrict__ task_kind, int64_t* __restrict__ cnt,
                                                const int64_t* __restrict__ off, Out O, unsigned long long* err,
                                                const int32_t* __restrict__ task_ord = nullptr) {
  GRID_LOOP(it, ntask) {
    // single pass: tasks visited grouped by kind (faces, edges, points), so a
    // warp runs one branch; records are keyed by the task's reference index t
    const int64_t t = task_ord ? (int64_t)task_ord[it] : it;
    const int st = task_st[t];
    const int kind = task_kind[t];
    const int feat = task_feat[t];
    const int32_t* sid = A.stris + 3 * st;
    const d3 s[3] = {ld3(A.x, sid[0]), ld3(A.x, sid[1]), ld3(A.x, sid[2])};
    int64_t c = 0;
    const int64_t base = Mode == 1 ? off[t] : (Mode == 2 ? t : 0);
    bool bad = false, ferr = false;
    Frame f;
    if (!tangent_frame(s[0], s[1], s[2], f)) {
      bad = true;
    } else if (kind == kFace) {  // sample_face, contact_sampling.hpp:97-141
      const int32_t* mid = A.mtris + 3 * feat;
      const d3 m[3] = {ld3(A.x, mid[0]), ld3(A.x, mid[1]), ld3(A.x, mid[2])};
      const d2 s2[3] = {to_plane(f, s[0]), to_plane(f, s[1]), to_plane(f, s[2])};
      const d2 m2[3] = {to_plane(f, m[0]), to_plane(f, m[1]), to_plane(f, m[2])};
      const double scale = local_scale(s);
      const double merge_tol = 1e-12 * scale;
      const double area_tol = 1e-14 * scale * scale;
      const double m_area = signed_area_2d(m2[0], m2[1], m2[2]);
      if (fabs(m_area) > area_tol) {
        d2 poly[12] = {m2[0], m2[1], m2[2]};
        if (m_area < 0) {
          const d2 tmp = poly[1];
          poly[1] = poly[2];
          poly[2] = tmp;
        }
        int n = clip_polygon(poly, 3, s2);
        n = merge_close(poly, n, merge_tol);
        if (n >= 3 && polygon_area(poly, n) > area_tol) {
          double q[6][4];
          const int nq = tri_quad(A.P.quad_order_face, q);
          for (int i = 1; i + 1 < n && !bad; ++i) {
            const d2 p0 = poly[0], p1 = poly[i], p2 = poly[i + 1];
            const double sub_area = signed_area_2d(p0, p1, p2);
            if (sub_area <= area_tol) continue;
            for (int k = 0; k < nq; ++k) {
              const d2 pt = (q[k][0] * p0 + q[k][1] * p1) + q[k][2] * p2;
              SampleRec r;
              r.type = GMCP_FACE;
              d3 bs;
              if (!barycentric_2d(pt, s2[0], s2[1], s2[2], bs) || !barycentric_2d(pt, m2[0], m2[1], m2[2], r.bm)) {
                bad = true;
                break;
              }
              r.bs = clamp_bary(bs);
              r.weight = q[k][3] * sub_area;
              r.gamma = hermite_step(min3(r.bm), A.P.delta_face);
              r.eta = 0;
              const d3 xs = (r.bs.x * s[0] + r.bs.y * s[1]) + r.bs.z * s[2];
              const d3 xm = (r.bm.x * m[0] + r.bm.y * m[1]) + r.bm.z * m[2];
              r.g = dot(f.n, xm - xs);
              r.master[0] = mid[0];
              r.master[1] = mid[1];
              r.master[2] = mid[2];
              put<Mode>(A, sid, r, c, base, O, ferr);
              if (ferr) {
                bad = true;
                break;
              }
            }
          }
        }
      }
    } else if (kind == kEdge) {  // sample_edge, contact_sampling.hpp:146-192
      const int32_t* eid = A.medges + 2 * feat;
      const d3 e0 = ld3(A.x, eid[0]), e1 = ld3(A.x, eid[1]);
      const d2 s2[3] = {to_plane(f, s[0]), to_plane(f, s[1]), to_plane(f, s[2])};
      const double scale = local_scale(s);
      const d2 q0 = to_plane(f, e0);
      const d2 dq = to_plane(f, e1) - q0;
      bool keep = !(norm2(dq) <= 1e-12 * scale);
      double t0 = 0, t1 = 1;
      for (int k = 0; k < 3 && keep; ++k) {
        const d2 a = s2[k];
        const d2 dir = s2[(k + 1) % 3] - a;
        const double ca = cross2(dir, q0 - a);
        const double dc = cross2(dir, dq);
        if (fabs(dc) <= 1e-14 * scale * scale) {
          if (ca < 0) keep = false;
        } else if (dc > 0) {
          t0 = dmax(t0, -ca / dc);
        } else {
          t1 = dmin(t1, -ca / dc);
        }
      }
      if (keep && (t1 - t0 > 1e-12)) {
        const double len3 = norm(e1 - e0) * (t1 - t0);
        double q[5][2];
        const int nq = seg_quad(A.P.quad_order_edge, q);
        for (int k = 0; k < nq; ++k) {
          SampleRec r;
          r.type = GMCP_EDGE;
          const double eta = t0 + (t1 - t0) * q[k][0];
          r.eta = eta;
          d3 bs;
          if (!barycentric_2d(q0 + eta * dq, s2[0], s2[1], s2[2], bs)) {
            bad = true;
            break;
          }
          r.bs = clamp_bary(bs);
          r.bm = mk3(0, 0, 0);
          r.weight = q[k][1] * len3;
          r.gamma = hermite_step(eta, A.P.delta_edge) * hermite_step(1.0 - eta, A.P.delta_edge);
          const d3 xs = (r.bs.x * s[0] + r.bs.y * s[1]) + r.bs.z * s[2];
          const d3 xm = (1.0 - eta) * e0 + eta * e1;
          r.g = dot(f.n, xm - xs);
          r.master[0] = eid[0];
          r.master[1] = eid[1];
          r.master[2] = -1;
          put<Mode>(A, sid, r, c, base, O, ferr);
          if (ferr) {
            bad = true;
            break;
          }
        }
      }
    } else {  // sample_point, contact_sampling.hpp:196-215
      const int vid = A.mverts[feat];
      const d3 v = ld3(A.x, vid);
      d3 bary;
      if (!barycentric_2d(to_plane(f, v), to_plane(f, s[0]), to_plane(f, s[1]), to_plane(f, s[2]), bary)) {
        bad = true;
      } else if (!(min3(bary) < -1e-12)) {
        SampleRec r;
        r.type = GMCP_POINT;
        r.bs = clamp_bary(bary);
        r.bm = mk3(0, 0, 0);
        r.eta = 0;
        r.weight = 1;
        r.gamma = 1;
        const d3 xs = (r.bs.x * s[0] + r.bs.y * s[1]) + r.bs.z * s[2];
        r.g = dot(f.n, v - xs);
        r.master[0] = vid;
        r.master[1] = r.master[2] = -1;
        put<Mode>(A, sid, r, c, base, O, ferr);
        if (ferr) bad = true;
      }
    }
    if (bad) atomicMin(err, (unsigned long long)t + 1);  // +1: 0 is reserved for ownership errors
    if (!Mode) cnt[t] = c;
  }
}

// Two-phase face sampling (sample_face, contact_sampling.hpp:97-141). Phase 1,
// one thread per face task: clip the projected master triangle against the
// slave triangle; a task whose clipped polygon survives (n >= 3 vertices,
// area above tol; a triangle clipped by a triangle has at most 6) appends
// (task, n, polygon) at a warp-aggregated slot. Phase 2, one thread per
// (polygon, fan sub-triangle): its quadrature points, keyed (task << 5 |
// (sub-triangle - 1) nq + point) -- the reference order after the sort. Every
// lane of a warp runs the same loop, unlike the one-thread-per-task kernel,
// where a warp waited on its longest polygon.
constexpr int kPolyMax = 6;
struct FacePoly {
  int32_t task, n;
  d2 v[kPolyMax];
};
__global__ void __launch_bounds__(128) k_face_clip(SamplerArgs A, int64_t nface, const int32_t* __restrict__ task_ord,
                                                   const int32_t* __restrict__ task_st,
                                                   const int32_t* __restrict__ task_feat, FacePoly* __restrict__ polys,
                                                   int64_t* __restrict__ subs, unsigned int* __restrict__ npoly,
                                                   int64_t cap, unsigned long long* err) {
  GRID_LOOP(it, nface) {
    const int64_t t = task_ord[it];
    const int st = task_st[t];
    const int32_t* sid = A.stris + 3 * st;
    const d3 s[3] = {ld3(A.x, sid[0]), ld3(A.x, sid[1]), ld3(A.x, sid[2])};
    Frame f;
    bool keep = false, bad = false;
    d2 poly[12];
    int n = 0;
    if (!tangent_frame(s[0], s[1], s[2], f)) {
      bad = true;
    } else {
      const int32_t* mid = A.mtris + 3 * task_feat[t];
      const d3 m[3] = {ld3(A.x, mid[0]), ld3(A.x, mid[1]), ld3(A.x, mid[2])};
      const d2 s2[3] = {to_plane(f, s[0]), to_plane(f, s[1]), to_plane(f, s[2])};
      const d2 m2[3] = {to_plane(f, m[0]), to_plane(f, m[1]), to_plane(f, m[2])};
      const double scale = local_scale(s);
      const double merge_tol = 1e-12 * scale;
      const double area_tol = 1e-14 * scale * scale;
      const double m_area = signed_area_2d(m2[0], m2[1], m2[2]);
      if (fabs(m_area) > area_tol) {
        poly[0] = m2[0];
        poly[1] = m2[1];
        poly[2] = m2[2];
        if (m_area < 0) {
          const d2 tmp = poly[1];
          poly[1] = poly[2];
          poly[2] = tmp;
        }
        n = clip_polygon(poly, 3, s2);
        n = merge_close(poly, n, merge_tol);
        keep = n >= 3 && polygon_area(poly, n) > area_tol;
        if (keep && n > kPolyMax) bad = true;  // cannot happen for two triangles
      }
    }
    if (bad) atomicMin(err, (unsigned long long)t + 1);
    keep = keep && !bad;
    const unsigned am = __ballot_sync(__activemask(), keep);
    if (keep) {
      const int lane = threadIdx.x & 31, leader = __ffs(am) - 1;
      unsigned lt;
      asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
      unsigned b0 = 0;
      if (lane == leader) b0 = atomicAdd(npoly, (unsigned)__popc(am));
      b0 = __shfl_sync(am, b0, leader);
      const int64_t i = (int64_t)b0 + __popc(am & lt);
      if (i < cap) {
        polys[i].task = (int32_t)t;
        polys[i].n = n;
        for (int k = 0; k < n; ++k) polys[i].v[k] = poly[k];
        subs[i] = n - 2;
      }
    }
  }
}
__global__ void __launch_bounds__(128) k_face_samples(SamplerArgs A, int64_t nsub, const int64_t* __restrict__ sub_off,
                                                      int64_t npoly, const FacePoly* __restrict__ polys,
                                                      const int32_t* __restrict__ task_st,
                                                      const int32_t* __restrict__ task_feat, Out O,
                                                      unsigned long long* err) {
  GRID_LOOP(j, nsub) {
    int64_t lo = 0, hi = npoly;  // polygon of sub-triangle j: last sub_off[p] <= j
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (sub_off[mid] <= j) lo = mid; else hi = mid;
    }
    const FacePoly& P = polys[lo];
    const int i = 1 + (int)(j - sub_off[lo]);  // fan sub-triangle (poly[0], poly[i], poly[i+1])
    const int64_t t = P.task;
    const int32_t* sid = A.stris + 3 * task_st[t];
    const d3 s[3] = {ld3(A.x, sid[0]), ld3(A.x, sid[1]), ld3(A.x, sid[2])};
    Frame f;
    tangent_frame(s[0], s[1], s[2], f);  // phase 1 checked it
    const int32_t* mid = A.mtris + 3 * task_feat[t];
    const d3 m[3] = {ld3(A.x, mid[0]), ld3(A.x, mid[1]), ld3(A.x, mid[2])};
    const d2 s2[3] = {to_plane(f, s[0]), to_plane(f, s[1]), to_plane(f, s[2])};
    const d2 m2[3] = {to_plane(f, m[0]), to_plane(f, m[1]), to_plane(f, m[2])};
    const double scale = local_scale(s);
    const double area_tol = 1e-14 * scale * scale;
    const d2 p0 = P.v[0], p1 = P.v[i], p2 = P.v[i + 1];
    const double sub_area = signed_area_2d(p0, p1, p2);
    if (sub_area <= area_tol) continue;
    double q[6][4];
    const int nq = tri_quad(A.P.quad_order_face, q);
    int64_t c = 0;
    bool bad = false, ferr = false;
    for (int k = 0; k < nq; ++k) {
      const d2 pt = (q[k][0] * p0 + q[k][1] * p1) + q[k][2] * p2;
      SampleRec r;
      r.type = GMCP_FACE;
      d3 bs;
      if (!barycentric_2d(pt, s2[0], s2[1], s2[2], bs) || !barycentric_2d(pt, m2[0], m2[1], m2[2], r.bm)) {
        bad = true;
        break;
      }
      r.bs = clamp_bary(bs);
      r.weight = q[k][3] * sub_area;
      r.gamma = hermite_step(min3(r.bm), A.P.delta_face);
      r.eta = 0;
      const d3 xs = (r.bs.x * s[0] + r.bs.y * s[1]) + r.bs.z * s[2];
      const d3 xm = (r.bm.x * m[0] + r.bm.y * m[1]) + r.bm.z * m[2];
      r.g = dot(f.n, xm - xs);
      r.master[0] = mid[0];
      r.master[1] = mid[1];
      r.master[2] = mid[2];
      put<2>(A, sid, r, c, t, O, ferr, (i - 1) * nq + k);
      if (ferr) {
        bad = true;
        break;
      }
    }
    if (bad) atomicMin(err, (unsigned long long)t + 1);
  }
}

// tasks per slave tri in reference order: faces (cand tris), edges (cand
// edges), points (owned vertices ascending); task_ord lists them grouped by
// kind (faces, edges, points). One thread per task: a binary search over the
// per-slave-tri offsets of its kind finds its slave tri.
__device__ __forceinline__ int32_t owner_of(const int64_t* __restrict__ off, int32_t nst, int64_t i) {
  int32_t lo = 0, hi = nst;  // last st with off[st] <= i
  while (hi - lo > 1) {
    const int32_t mid = (lo + hi) >> 1;
    if (off[mid] <= i) lo = mid; else hi = mid;
  }
  return lo;
}
__global__ void k_tasks(int32_t nst, const int64_t* __restrict__ toff, const int32_t* __restrict__ tids,
                        const int64_t* __restrict__ eoff, const int32_t* __restrict__ eids,
                        const int64_t* __restrict__ poff, const int32_t* __restrict__ pids,
                        int32_t* __restrict__ task_st, int32_t* __restrict__ task_feat, int8_t* __restrict__ task_kind,
                        int32_t* __restrict__ task_ord) {
  const int64_t nf = toff[nst], ne = eoff[nst], np = poff[nst];
  GRID_LOOP(g, nf + ne + np) {
    int kind;
    int64_t i;
    const int64_t* off;
    if (g < nf) { kind = kFace; i = g; off = toff; }
    else if (g < nf + ne) { kind = kEdge; i = g - nf; off = eoff; }
    else { kind = kPoint; i = g - nf - ne; off = poff; }
    const int32_t st = owner_of(off, nst, i);
    // reference index: the slave tri's earlier tasks, then this kind's earlier ones
    const int64_t base = toff[st] + eoff[st] + poff[st];
    const int64_t o = base + (kind == kFace ? i - toff[st]
                                            : kind == kEdge ? (toff[st + 1] - toff[st]) + (i - eoff[st])
                                                            : (toff[st + 1] - toff[st]) + (eoff[st + 1] - eoff[st]) +
                                                                  (i - poff[st]));
    task_st[o] = st;
    task_feat[o] = kind == kFace ? tids[i] : kind == kEdge ? eids[i] : pids[i];
    task_kind[o] = (int8_t)kind;
    task_ord[g] = (int32_t)o;
  }
}

__global__ void k_iota(int64_t n, uint32_t* __restrict__ v) {
  GRID_LOOP(i, n) v[i] = (uint32_t)i;
}

// single-pass sampler: staged records -> reference order (sorted keys)
__global__ void k_unstage(int64_t n, const uint32_t* __restrict__ src_of, Out S, Out O) {
  GRID_LOOP(i, n) {
    const int64_t j = src_of[i];
    O.type[i] = S.type[j];
    for (int k = 0; k < 3; ++k) {
      O.slave[3 * i + k] = S.slave[3 * j + k];
      O.master[3 * i + k] = S.master[3 * j + k];
      O.beta_s[3 * i + k] = S.beta_s[3 * j + k];
      O.beta_m[3 * i + k] = S.beta_m[3 * j + k];
    }
    O.eta[i] = S.eta[j];
    O.weight[i] = S.weight[j];
    O.gamma[i] = S.gamma[j];
    O.eps[i] = S.eps[j];
    O.g_ref[i] = S.g_ref[j];
  }
}

// CSR offsets from sorted keys whose high 32 bits are the segment id.
__global__ void k_seg_offsets(int64_t n, const unsigned long long* __restrict__ keys, int32_t nseg,
                              int64_t* __restrict__ off) {
  GRID_LOOP(s, (int64_t)nseg + 1) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if ((int64_t)(keys[mid] >> 32) < s) lo = mid + 1; else hi = mid;
    }
    off[s] = lo;
  }
}
__global__ void k_low32(int64_t n, const unsigned long long* __restrict__ keys, int32_t* __restrict__ out) {
  GRID_LOOP(i, n) out[i] = (int32_t)(keys[i] & 0xffffffffull);
}
__global__ void k_pair_keys(int32_t nst, const int64_t* __restrict__ off, const int32_t* __restrict__ ids,
                            unsigned long long* __restrict__ keys) {
  GRID_LOOP(st, nst) {
    for (int64_t i = off[st]; i < off[st + 1]; ++i) keys[i] = ((unsigned long long)ids[i] << 32) | (unsigned int)st;
  }
}

int64_t last_of(const DBuf<int64_t>& a, int64_t idx, cudaStream_t s) {
  int64_t v = 0;
  GMCP_CUDA(cudaMemcpyAsync(&v, a.p + idx, sizeof v, cudaMemcpyDeviceToHost, s));
  GMCP_CUDA(cudaStreamSynchronize(s));
  return v;
}

// ---------------------------------------------------------------------------
// Dual-mesh embedding (embedding.hpp:26-106)

// geometry.hpp:45-103: closest point on the closed triangle (Voronoi regions)
__device__ __forceinline__ d3 closest_point_on_triangle(d3 p, d3 a, d3 b, d3 c) {
  const d3 ab = b - a, ac = c - a, ap = p - a;
  const double d1 = dot(ab, ap), d2 = dot(ac, ap);
  if (d1 <= 0 && d2 <= 0) return a;
  const d3 bp = p - b;
  const double d3v = dot(ab, bp), d4 = dot(ac, bp);
  if (d3v >= 0 && d4 <= d3v) return b;
  const double vc = d1 * d4 - d3v * d2;
  if (vc <= 0 && d1 >= 0 && d3v <= 0) return a + (d1 / (d1 - d3v)) * ab;
  const d3 cp = p - c;
  const double d5 = dot(ab, cp), d6 = dot(ac, cp);
  if (d6 >= 0 && d5 <= d6) return c;
  const double vb = d5 * d2 - d1 * d6;
  if (vb <= 0 && d2 >= 0 && d6 <= 0) return a + (d2 / (d2 - d6)) * ac;
  const double va = d3v * d6 - d5 * d4;
  if (va <= 0 && (d4 - d3v) >= 0 && (d5 - d6) >= 0) return b + ((d4 - d3v) / ((d4 - d3v) + (d5 - d6))) * (c - b);
  const double denom = 1.0 / ((va + vb) + vc);
  const double v = vb * denom, w = vc * denom;
  return (a + v * ab) + w * ac;
}

__device__ __forceinline__ double box_sq_dist(const Box& b, d3 p) {  // core.hpp:86-89
  const double pv[3] = {p.x, p.y, p.z};
  double s = 0;
  for (int k = 0; k < 3; ++k) {
    const double d = dmax(dmax(b.lo[k] - pv[k], 0.0), pv[k] - b.hi[k]);
    s = k == 0 ? d * d : s + d * d;
  }
  return s;
}

// host triangle checks: exact-zero area (embedding.hpp:30-35, by index) and
// triangle_normal's area cutoff (closest_point_on_triangle would throw)
__global__ void k_embed_check(int32_t nt, const int32_t* __restrict__ tris, const double* __restrict__ x,
                              unsigned long long* bad) {
  GRID_LOOP(t, nt) {
    const d3 a = ld3(x, tris[3 * t]), b = ld3(x, tris[3 * t + 1]), c = ld3(x, tris[3 * t + 2]);
    if (!(norm(cross(b - a, c - a)) > 0)) atomicMin(&bad[0], (unsigned long long)t);
    d3 n;
    if (!triangle_normal(a, b, c, n)) atomicMin(&bad[1], (unsigned long long)t);
  }
}

// nearest host triangle (min squared distance, lowest index on ties) by LBVH
// branch and bound, then plane barycentrics and the normal offset
__global__ void k_embed(int64_t np, const double* __restrict__ pts, int32_t nt, const int32_t* __restrict__ tris,
                        const double* __restrict__ x, const Box* __restrict__ nodes, const int32_t* __restrict__ left,
                        const int32_t* __restrict__ right, const int32_t* __restrict__ sorted_idx,
                        int32_t* __restrict__ tri_out, double* __restrict__ bary, double* __restrict__ offset,
                        unsigned long long* bad) {
  GRID_LOOP(i, np) {
    const d3 p = ld3(pts, i);
    int best = -1;
    double best_d2 = kDblMax;
    int stack[64];
    int top = 0;
    stack[top++] = 0;
    while (top > 0) {
      const int node = stack[--top];
      // conservative prune: equal (or rounding-close) lower bounds are still
      // visited so index ties break exactly as a full scan would
      if (best >= 0 && box_sq_dist(nodes[node], p) > best_d2 * (1.0 + 1e-12) + 1e-300) continue;
      if (node >= nt - 1) {
        const int t = sorted_idx[node - (nt - 1)];
        const d3 a = ld3(x, tris[3 * t]), b = ld3(x, tris[3 * t + 1]), c = ld3(x, tris[3 * t + 2]);
        const d3 q = closest_point_on_triangle(p, a, b, c) - p;
        const double d2 = dot(q, q);
        if (d2 < best_d2 || (d2 == best_d2 && t < best)) {
          best_d2 = d2;
          best = t;
        }
      } else {
        if (top + 2 > 64) {
          atomicExch(&bad[2], 1ull);
          break;
        }
        stack[top++] = right[node];
        stack[top++] = left[node];
      }
    }
    const d3 a = ld3(x, tris[3 * best]), b = ld3(x, tris[3 * best + 1]), c = ld3(x, tris[3 * best + 2]);
    d3 n;
    triangle_normal(a, b, c, n);
    const d3 d = p - a, e1 = b - a, e2 = c - a;
    // geometry.hpp:26-34 solve_barycentric_gram
    const double a11 = dot(e1, e1), a12 = dot(e1, e2), a22 = dot(e2, e2);
    const double b1 = dot(d, e1), b2 = dot(d, e2);
    const double det = a11 * a22 - a12 * a12;
    if (!(det > 1e-14 * a11 * a22)) atomicMin(&bad[1], (unsigned long long)best);
    const double v = (a22 * b1 - a12 * b2) / det, w = (a11 * b2 - a12 * b1) / det;
    tri_out[i] = best;
    bary[3 * i] = (1.0 - v) - w;
    bary[3 * i + 1] = v;
    bary[3 * i + 2] = w;
    offset[i] = dot(n, d);
  }
}

// embedding.hpp:87-106; bad = first embedded vertex whose host triangle degenerated
__global__ void k_apply_embedding(int64_t n, const int32_t* __restrict__ tri, const double* __restrict__ bary,
                                  const double* __restrict__ offset, const int32_t* __restrict__ tris,
                                  const double* __restrict__ x, double* __restrict__ out, unsigned long long* bad) {
  GRID_LOOP(i, n) {
    const int32_t* t = tris + 3 * (int64_t)tri[i];
    const d3 v0 = ld3(x, t[0]), v1 = ld3(x, t[1]), v2 = ld3(x, t[2]);
    d3 nn;
    if (!triangle_normal(v0, v1, v2, nn)) {
      atomicMin(bad, (unsigned long long)i);
      continue;
    }
    const d3 r = ((bary[3 * i] * v0 + bary[3 * i + 1] * v1) + bary[3 * i + 2] * v2) + offset[i] * nn;
    out[3 * i] = r.x;
    out[3 * i + 1] = r.y;
    out[3 * i + 2] = r.z;
  }
}

// LBVH over triangles (K1): boxes, Morton keys (+ scene id for batches),
// radix sort, Karras hierarchy, bottom-up refit. Internal nodes 0..n-2,
// leaves n-1..2n-2 (leaf k -> triangle idx_sorted[k]).
struct Lbvh {
  DBuf<Box> tboxes, nodes;
  DBuf<unsigned long long> bounds, keys, keys_sorted;
  DBuf<int32_t> idx, idx_sorted, left, right, parent, flags;
  DBuf<int2> srange;  // per-node [min, max] scene (batched scenes only)
};

int lbvh_build(Lbvh& B, int32_t n, const int32_t* tris, const double* x, const int32_t* vsc, int n_scenes,
               cudaStream_t s) {
  B.tboxes.resize(n);
  B.bounds.resize(6);
  const unsigned long long binit[6] = {~0ull, ~0ull, ~0ull, 0, 0, 0};
  GMCP_CUDA(cudaMemcpyAsync(B.bounds.p, binit, sizeof binit, cudaMemcpyHostToDevice, s));
  k_master_boxes<<<grid_for(n, 256), 256, 0, s>>>(n, tris, x, B.tboxes.p, B.bounds.p);
  B.keys.resize(n);
  B.keys_sorted.resize(n);
  B.idx.resize(n);
  B.idx_sorted.resize(n);
  int ib = 32;  // index bits of the key; fewer when a scene id must fit above the Morton code
  if (vsc) {
    ib = 1;
    while ((1ll << ib) < n) ++ib;
    int sb = 1;
    while ((1 << sb) < n_scenes) ++sb;
    if (sb + 30 + ib > 64) throw StatusError(GMCP_ERR_CONFIG, "batched broadphase: too many scenes x triangles");
  }
  k_morton<<<grid_for(n, 256), 256, 0, s>>>(n, B.tboxes.p, B.bounds.p, tris, vsc, ib, B.keys.p, B.idx.p);
  sort_pairs(B.keys.p, B.keys_sorted.p, B.idx.p, B.idx_sorted.p, n, s, 64);
  const int nnodes = 2 * n - 1;
  B.nodes.resize(nnodes);
  B.left.resize(std::max(n - 1, 1));
  B.right.resize(std::max(n - 1, 1));
  B.parent.resize(nnodes);
  B.flags.resize(std::max(n - 1, 1));
  B.flags.zero(s);
  GMCP_CUDA(cudaMemsetAsync(B.parent.p, 0xff, nnodes * sizeof(int32_t), s));
  if (n > 1) k_karras<<<grid_for(n - 1, 256), 256, 0, s>>>(n, B.keys_sorted.p, B.left.p, B.right.p, B.parent.p);
  if (vsc) B.srange.resize(nnodes);
  k_refit<<<grid_for(n, 256), 256, 0, s>>>(n, B.idx_sorted.p, B.tboxes.p, B.left.p, B.right.p, B.parent.p, B.nodes.p,
                                           B.flags.p, tris, vsc, B.srange.p);
  return 3 + (n > 1 ? 1 : 0) + 2;
}

// Broadphase + sampler scratch kept per context across rebuilds (grow-only:
// no cudaMalloc / cudaFree on the rebuild path after the first one).
struct RebuildTmp : TmpBase {
  Lbvh bvh;
  DBuf<int64_t> cnt;
  DBuf<int> ovf, wovf;
  DBuf<int32_t> tmp_e, tmp_v;
  DBuf<int64_t> ecnt, vcnt;
  DBuf<unsigned long long> err;
  DBuf<unsigned long long> k1, k2;
  DBuf<int64_t> by_off, pcnt, poff, pt_off;
  DBuf<int32_t> by_st, pt_ids;
  DBuf<int32_t> task_st, task_feat, task_ord;
  DBuf<FacePoly> polys;
  DBuf<int64_t> poly_sub, sub_off;
  DBuf<unsigned int> npoly;
  DBuf<int8_t> task_kind;
  DBuf<int64_t> tcnt, toff;
  struct Stage {
    DBuf<int8_t> type;
    DBuf<int32_t> slave, master;
    DBuf<double> beta_s, beta_m, eta, weight, gamma, eps, gref;
  } stage;                        // single-pass sampler staging (unordered)
  int64_t stage_cap = 0;
  DBuf<uint32_t> skey, skey2, sidx, sidx2;
  DBuf<unsigned int> sctr;
};
RebuildTmp& rebuild_tmp(Ctx& c) {
  if (!c.rebuild_tmp) c.rebuild_tmp = std::make_unique<RebuildTmp>();
  return *static_cast<RebuildTmp*>(c.rebuild_tmp.get());
}

}  // namespace

// ===========================================================================

void run_broadphase(Ctx& c, double r, int64_t* counts) {
  const NvtxRange nvtx_("gmcp:K1-K3 broadphase");
  RebuildTmp& RT = rebuild_tmp(c);
  cudaStream_t s = c.stream;
  // self-contact check (contact_sampling.hpp:286-294), host mirrors are sorted
  {
    const auto& a = c.slave.h_verts;
    const auto& b = c.master.h_verts;
    size_t i = 0, j = 0;
    while (i < a.size() && j < b.size()) {
      if (a[i] == b[j])
        throw StatusError(GMCP_ERR_CONFIG,
                          "build_candidate_pairs: slave and master share vertices (self-contact is not supported)");
      if (a[i] < b[j]) ++i; else ++j;
    }
  }
  const int32_t nst = c.slave.n_tris, nmt = c.master.n_tris;
  for (int k = 0; k < 3; ++k) {
    c.pair_off[k].resize(nst + 1);
    c.pair_off[k].zero(s);
  }
  if (nst == 0 || nmt == 0) {
    for (int k = 0; k < 3; ++k) c.pair_ids[k].resize(0);
    c.have_pairs = true;
    counts[0] = counts[1] = counts[2] = 0;
    c.sync();
    return;
  }
  // K1: boxes, Morton keys, sort, hierarchy, refit
  const int32_t* vsc = c.vscene.n ? c.vscene.p : nullptr;
  if (vsc && (int64_t)c.vscene.n != c.n_vertices())
    throw StatusError(GMCP_ERR_CONFIG, "batched broadphase: vertex scene ids do not cover the positions");
  Lbvh& B = RT.bvh;
  c.launches += lbvh_build(B, nmt, c.master.tris.p, c.X(), vsc, c.n_scenes, s);
  auto& nodes = B.nodes;
  auto& left = B.left;
  auto& right = B.right;
  auto& idx_sorted = B.idx_sorted;
  auto& srange = B.srange;
  // K2: count, scan, emit+sort
  const uint8_t* smask = vsc && c.use_scene_mask ? c.scene_mask.p : nullptr;
  auto& tmp_e = RT.tmp_e;
  auto& tmp_v = RT.tmp_v;
  auto& ecnt = RT.ecnt;
  auto& vcnt = RT.vcnt;
  auto& cnt = RT.cnt;
  auto& ovf = RT.ovf;
  cnt.resize(nst + 1);
  cnt.zero(s);
  ovf.resize(1);
  ovf.zero(s);
  auto& wovf = RT.wovf;
  wovf.resize(1);
  // batched scenes keep the per-thread traversal: a scene-pruned query descends
  // a 1-2 node frontier through the packed tree's upper levels, where 32
  // independent queries per warp beat one query per warp
  bool warp_path = !c.thread_query && vsc == nullptr;
  bool warp_feat = warp_path;  // (the warp feature kernel on batched scenes: broadphase 4.6 -> 6.5 ms per C5 pass)
  for (;;) {  // the warp-cooperative kernels; the per-thread ones if a warp ran out of shared memory
    cnt.zero(s);
    wovf.zero(s);
    const int gq = (int)std::min<int64_t>((nst + kQW - 1) / kQW, 148 * 64);
    if (warp_path)
      k_query_warp<0><<<gq, 32 * kQW, 0, s>>>(nst, c.slave.tris.p, c.X(), r, nmt, nodes.p, left.p, right.p,
                                              idx_sorted.p, cnt.p, nullptr, nullptr, wovf.p, vsc, srange.p, smask);
    else
      k_query<0><<<grid_for(nst, 128), 128, 0, s>>>(nst, c.slave.tris.p, c.X(), r, nmt, nodes.p, left.p, right.p,
                                                     idx_sorted.p, cnt.p, nullptr, nullptr, ovf.p, vsc, srange.p,
                                                     smask);
    exclusive_scan(cnt.p, c.pair_off[0].p, nst + 1, s);
    const int64_t ntri = last_of(c.pair_off[0], nst, s);
    c.pair_ids[0].resize(std::max<int64_t>(ntri, 1));
    if (warp_path)
      k_query_warp<1><<<gq, 32 * kQW, 0, s>>>(nst, c.slave.tris.p, c.X(), r, nmt, nodes.p, left.p, right.p,
                                              idx_sorted.p, nullptr, c.pair_off[0].p, c.pair_ids[0].p, wovf.p, vsc,
                                              srange.p, smask);
    else
      k_query<1><<<grid_for(nst, 128), 128, 0, s>>>(nst, c.slave.tris.p, c.X(), r, nmt, nodes.p, left.p, right.p,
                                                     idx_sorted.p, nullptr, c.pair_off[0].p, c.pair_ids[0].p, ovf.p,
                                                     vsc, srange.p, smask);
    c.pair_ids[0].n = ntri;
    // K3: candidate edges / verts
    tmp_e.resize(std::max<int64_t>(3 * ntri, 1));
    tmp_v.resize(std::max<int64_t>(3 * ntri, 1));
    ecnt.resize(nst + 1);
    vcnt.resize(nst + 1);
    ecnt.zero(s);
    vcnt.zero(s);
    if (warp_feat)
      k_features_warp<<<gq, 32 * kQW, 0, s>>>(nst, c.pair_off[0].p, c.pair_ids[0].p, c.master.tris.p,
                                              c.master.tri_edges.p, c.master.verts.p, c.master.n_verts, tmp_e.p,
                                              tmp_v.p, ecnt.p, vcnt.p, wovf.p);
    else
      k_features<<<grid_for(nst, 128), 128, 0, s>>>(nst, c.pair_off[0].p, c.pair_ids[0].p, c.master.tris.p,
                                                     c.master.tri_edges.p, c.master.verts.p, c.master.n_verts,
                                                     tmp_e.p, tmp_v.p, ecnt.p, vcnt.p);
    c.launches += 3;
    if (!warp_path && !warp_feat) break;
    int wo = 0;
    GMCP_CUDA(cudaMemcpyAsync(&wo, wovf.p, sizeof wo, cudaMemcpyDeviceToHost, s));
    c.sync();
    if (!wo) break;
    warp_path = warp_feat = false;
  }
  exclusive_scan(ecnt.p, c.pair_off[1].p, nst + 1, s);
  exclusive_scan(vcnt.p, c.pair_off[2].p, nst + 1, s);
  const int64_t ne = last_of(c.pair_off[1], nst, s), nv = last_of(c.pair_off[2], nst, s);
  c.pair_ids[1].resize(std::max<int64_t>(ne, 1));
  c.pair_ids[2].resize(std::max<int64_t>(nv, 1));
  k_compact<<<grid_for(nst, 128), 128, 0, s>>>(nst, c.pair_off[0].p, tmp_e.p, c.pair_off[1].p, c.pair_ids[1].p);
  k_compact<<<grid_for(nst, 128), 128, 0, s>>>(nst, c.pair_off[0].p, tmp_v.p, c.pair_off[2].p, c.pair_ids[2].p);
  c.pair_ids[1].n = ne;
  c.pair_ids[2].n = nv;
  c.launches += 2;
  const int64_t ntri = c.pair_ids[0].n;
  GMCP_CUDA(cudaGetLastError());
  int of = 0;
  GMCP_CUDA(cudaMemcpyAsync(&of, ovf.p, sizeof of, cudaMemcpyDeviceToHost, s));
  c.sync();
  if (of) throw StatusError(GMCP_ERR_CONFIG, "broadphase: LBVH traversal stack overflow");
  counts[0] = ntri;
  counts[1] = ne;
  counts[2] = nv;
  c.have_pairs = true;
}

int64_t run_sampler(Ctx& c, const double* eps_ref_dev) {
  const NvtxRange nvtx_("gmcp:K4-K5 sampler");
  RebuildTmp& RT = rebuild_tmp(c);
  cudaStream_t s = c.stream;
  const int32_t nst = c.slave.n_tris, nmv = c.master.n_verts;
  SamplerArgs A;
  A.x = c.X();
  A.eps_ref = eps_ref_dev;
  A.nst = nst;
  A.stris = c.slave.tris.p;
  A.mtris = c.master.tris.p;
  A.medges = c.master.edges.p;
  A.mverts = c.master.verts.p;
  A.P = c.params;
  auto& err = RT.err;
  err.resize(1);
  GMCP_CUDA(cudaMemsetAsync(err.p, 0xff, sizeof(unsigned long long), s));

  // K4: inverse lists mv -> slave tris (ascending st), ownership, regroup by st
  const int64_t nvc = (int64_t)c.pair_ids[2].n;
  auto& k1 = RT.k1;
  auto& k2 = RT.k2;
  auto& by_off = RT.by_off;
  auto& pcnt = RT.pcnt;
  auto& poff = RT.poff;
  auto& pt_off = RT.pt_off;
  auto& by_st = RT.by_st;
  auto& pt_ids = RT.pt_ids;
  by_off.resize(nmv + 1);
  by_st.resize(std::max<int64_t>(nvc, 1));
  if (nvc) {
    k1.resize(nvc);
    k2.resize(nvc);
    k_pair_keys<<<grid_for(nst, 128), 128, 0, s>>>(nst, c.pair_off[2].p, c.pair_ids[2].p, k1.p);
    sort_keys(k1.p, k2.p, nvc, s, 64);
    k_seg_offsets<<<grid_for(nmv + 1, 256), 256, 0, s>>>(nvc, k2.p, nmv, by_off.p);
    k_low32<<<grid_for(nvc, 256), 256, 0, s>>>(nvc, k2.p, by_st.p);
    c.launches += 3;
  } else {
    by_off.zero(s);
  }
  pcnt.resize(nmv + 1);
  pcnt.zero(s);
  poff.resize(nmv + 1);
  if (nmv) {
    k_point_owner<0><<<grid_for(nmv, 128), 128, 0, s>>>(A, nmv, by_off.p, by_st.p, pcnt.p, nullptr, nullptr, err.p);
    ++c.launches;
  }
  exclusive_scan(pcnt.p, poff.p, nmv + 1, s);
  const int64_t npts = last_of(poff, nmv, s);
  pt_off.resize(nst + 1);
  pt_ids.resize(std::max<int64_t>(npts, 1));
  if (npts) {
    k1.resize(npts);
    k2.resize(npts);
    k_point_owner<1><<<grid_for(nmv, 128), 128, 0, s>>>(A, nmv, by_off.p, by_st.p, nullptr, poff.p, k1.p, err.p);
    sort_keys(k1.p, k2.p, npts, s, 64);
    k_seg_offsets<<<grid_for(nst + 1, 256), 256, 0, s>>>(npts, k2.p, nst, pt_off.p);
    k_low32<<<grid_for(npts, 256), 256, 0, s>>>(npts, k2.p, pt_ids.p);
    c.launches += 3;
  } else {
    pt_off.zero(s);
  }
  // K5: tasks in reference order, count -> scan -> emit
  const int64_t ntask = (int64_t)c.pair_ids[0].n + (int64_t)c.pair_ids[1].n + npts;
  auto& task_st = RT.task_st;
  auto& task_feat = RT.task_feat;
  auto& task_kind = RT.task_kind;
  auto& tcnt = RT.tcnt;
  auto& toff = RT.toff;
  task_st.resize(std::max<int64_t>(ntask, 1));
  task_feat.resize(std::max<int64_t>(ntask, 1));
  task_kind.resize(std::max<int64_t>(ntask, 1));
  RT.task_ord.resize(std::max<int64_t>(ntask, 1));
  static const bool kind_order = !std::getenv("GMCP_SAMPLER_TASK_ORDER") || std::atoi(std::getenv("GMCP_SAMPLER_TASK_ORDER")) != 0;
  Out O{};
  if (ntask) {
    k_tasks<<<grid_for(ntask, 256), 256, 0, s>>>(nst, c.pair_off[0].p, c.pair_ids[0].p, c.pair_off[1].p,
                                                c.pair_ids[1].p, pt_off.p, pt_ids.p, task_st.p, task_feat.p,
                                                task_kind.p, RT.task_ord.p);
    ++c.launches;
  }
  if (ntask >= (int64_t)1 << 27) throw StatusError(GMCP_ERR_CONFIG, "sampler: too many (slave tri, feature) tasks");
  // one pass over the tasks: every accepted sample goes to a staging slot
  // (warp-aggregated atomics) keyed by (task, index in task); a radix sort of
  // the keys then restores the reference order (contact_sampling.hpp:438-468)
  auto& st_ = RT.stage;
  auto& skey = RT.skey;
  auto& skey2 = RT.skey2;
  auto& sidx = RT.sidx;
  auto& sidx2 = RT.sidx2;
  auto& sctr = RT.sctr;
  sctr.resize(1);
  // face tasks (the first nface of the kind order): two-phase sampling
  int64_t nface_done = 0, npoly = 0, nsub = 0;
  static const bool face_split =
      !std::getenv("GMCP_SAMPLER_FACE_SPLIT") || std::atoi(std::getenv("GMCP_SAMPLER_FACE_SPLIT")) != 0;
  if (kind_order && face_split && ntask) {
    const int64_t nface = c.pair_ids[0].n;
    RT.polys.resize(std::max<int64_t>(nface, 1));
    RT.poly_sub.resize(nface + 1);
    RT.sub_off.resize(nface + 1);
    RT.npoly.resize(1);
    RT.npoly.zero(s);
    if (nface) {
      k_face_clip<<<grid_for(nface, 128), 128, 0, s>>>(A, nface, RT.task_ord.p, task_st.p, task_feat.p, RT.polys.p,
                                                       RT.poly_sub.p, RT.npoly.p, nface, err.p);
      ++c.launches;
    }
    unsigned int np_h = 0;
    GMCP_CUDA(cudaMemcpyAsync(&np_h, RT.npoly.p, sizeof np_h, cudaMemcpyDeviceToHost, s));
    c.sync();
    npoly = np_h;
    if (npoly) {
      GMCP_CUDA(cudaMemsetAsync(RT.poly_sub.p + npoly, 0, sizeof(int64_t), s));
      exclusive_scan(RT.poly_sub.p, RT.sub_off.p, npoly + 1, s);
      nsub = last_of(RT.sub_off, npoly, s);
    }
    nface_done = nface;
  }
  int64_t cap = std::max<int64_t>({RT.stage_cap, ntask, c.ns + c.ns / 4, 1});
  unsigned int cnt_h = 0;
  for (int attempt = 0; attempt < 2; ++attempt) {
    if (cap > RT.stage_cap) {
      st_.type.resize(cap);
      st_.slave.resize(3 * cap);
      st_.master.resize(3 * cap);
      st_.beta_s.resize(3 * cap);
      st_.beta_m.resize(3 * cap);
      st_.eta.resize(cap);
      st_.weight.resize(cap);
      st_.gamma.resize(cap);
      st_.eps.resize(cap);
      st_.gref.resize(cap);
      skey.resize(cap);
      RT.stage_cap = cap;
    }
    Out SO{st_.type.p, st_.slave.p, st_.master.p, st_.beta_s.p, st_.beta_m.p, st_.eta.p,
           st_.weight.p, st_.gamma.p, st_.eps.p, st_.gref.p, skey.p, sctr.p, cap};
    sctr.zero(s);
    if (nsub > 0) {
      k_face_samples<<<grid_for(nsub, 128), 128, 0, s>>>(A, nsub, RT.sub_off.p, npoly, RT.polys.p, task_st.p,
                                                          task_feat.p, SO, err.p);
      ++c.launches;
    }
    if (ntask - nface_done > 0) {
      k_sample<2><<<grid_for(ntask - nface_done, 128), 128, 0, s>>>(
          A, ntask - nface_done, task_st.p, task_feat.p, task_kind.p, nullptr, nullptr, SO, err.p,
          kind_order ? RT.task_ord.p + nface_done : nullptr);
      ++c.launches;
    }
    GMCP_CUDA(cudaMemcpyAsync(&cnt_h, sctr.p, sizeof cnt_h, cudaMemcpyDeviceToHost, s));
    c.sync();
    if ((int64_t)cnt_h <= cap) break;
    cap = (int64_t)cnt_h;  // staging was too small: every record counted, re-run with room
  }
  const int64_t n = cnt_h;
  unsigned long long e = 0;
  GMCP_CUDA(cudaMemcpyAsync(&e, err.p, sizeof e, cudaMemcpyDeviceToHost, s));
  c.sync();
  if (e != ~0ull) throw StatusError(GMCP_ERR_DEGENERATE, "build_contact_state: degenerate triangle (MeshError)");
  c.ns = n;
  c.s_type.resize(n);
  c.s_slave.resize(3 * n);
  c.s_master.resize(3 * n);
  c.s_beta_s.resize(3 * n);
  c.s_beta_m.resize(3 * n);
  c.s_eta.resize(n);
  c.s_weight.resize(n);
  c.s_gamma.resize(n);
  c.s_eps.resize(n);
  c.s_gref.resize(n);
  O = Out{c.s_type.p, c.s_slave.p, c.s_master.p, c.s_beta_s.p, c.s_beta_m.p, c.s_eta.p,
          c.s_weight.p, c.s_gamma.p, c.s_eps.p, c.s_gref.p};
  if (n) {
    skey2.resize(n);
    sidx.resize(n);
    sidx2.resize(n);
    k_iota<<<grid_for(n, 256), 256, 0, s>>>(n, sidx.p);
    int kb = 5;
    while (((int64_t)1 << kb) < (ntask << 5)) ++kb;
    sort_pairs(skey.p, skey2.p, sidx.p, sidx2.p, n, s, kb);
    Out SO{st_.type.p, st_.slave.p, st_.master.p, st_.beta_s.p, st_.beta_m.p, st_.eta.p,
           st_.weight.p, st_.gamma.p, st_.eps.p, st_.gref.p};
    k_unstage<<<grid_for(n, 256), 256, 0, s>>>(n, sidx2.p, SO, O);
    c.launches += 2;
  }
  GMCP_CUDA(cudaGetLastError());
  derive_sample_fields(c);
  c.sync();
  return n;
}

// ===========================================================================
// embedding host entry points (embedding.hpp:26-106)

struct EmbedTmp : TmpBase {
  Lbvh bvh;
  DBuf<double> pts, x, bary, off, out;
  DBuf<int32_t> tris, tri;
  DBuf<unsigned long long> bad;
};
static EmbedTmp& embed_tmp(Ctx& c) {
  if (!c.embed_tmp) c.embed_tmp = std::make_unique<EmbedTmp>();
  return *static_cast<EmbedTmp*>(c.embed_tmp.get());
}

void run_embed(Ctx& c, const double* points, int64_t np, const double* host_v, int64_t nhv, const int32_t* host_t,
               int64_t nht, int32_t* tri, double* bary, double* offset, int64_t* bad) {
  cudaStream_t s = c.stream;
  *bad = -1;
  if (nht <= 0) throw StatusError(GMCP_ERR_CONFIG, "embedding host has no triangles");
  if (nht >= (int64_t)INT32_MAX / 2) throw StatusError(GMCP_ERR_CONFIG, "embedding host too large");
  EmbedTmp& E = embed_tmp(c);
  E.x.upload(host_v, 3 * nhv, s);
  E.tris.upload(host_t, 3 * nht, s);
  E.bad.resize(3);
  const unsigned long long binit[3] = {~0ull, ~0ull, 0};
  GMCP_CUDA(cudaMemcpyAsync(E.bad.p, binit, sizeof binit, cudaMemcpyHostToDevice, s));
  const int32_t nt = (int32_t)nht;
  k_embed_check<<<grid_for(nt, 256), 256, 0, s>>>(nt, E.tris.p, E.x.p, E.bad.p);
  ++c.launches;
  unsigned long long h[3];
  GMCP_CUDA(cudaMemcpyAsync(h, E.bad.p, sizeof h, cudaMemcpyDeviceToHost, s));
  c.sync();
  if (h[0] != ~0ull) {
    *bad = (int64_t)h[0];
    throw StatusError(GMCP_ERR_DEGENERATE, "embedding host triangle " + std::to_string(h[0]) + " is degenerate",
                      (int64_t)h[0]);
  }
  if (h[1] != ~0ull)
    throw StatusError(GMCP_ERR_DEGENERATE, "triangle_normal: degenerate triangle (area below cutoff)");
  if (np == 0) return;
  c.launches += lbvh_build(E.bvh, nt, E.tris.p, E.x.p, nullptr, 1, s);
  E.pts.upload(points, 3 * np, s);
  E.tri.resize(np);
  E.bary.resize(3 * np);
  E.off.resize(np);
  k_embed<<<grid_for(np, 128), 128, 0, s>>>(np, E.pts.p, nt, E.tris.p, E.x.p, E.bvh.nodes.p, E.bvh.left.p,
                                             E.bvh.right.p, E.bvh.idx_sorted.p, E.tri.p, E.bary.p, E.off.p, E.bad.p);
  ++c.launches;
  GMCP_CUDA(cudaGetLastError());
  GMCP_CUDA(cudaMemcpyAsync(h, E.bad.p, sizeof h, cudaMemcpyDeviceToHost, s));
  E.tri.download(tri, np, s);
  E.bary.download(bary, 3 * np, s);
  E.off.download(offset, np, s);
  c.sync();
  if (h[2]) throw StatusError(GMCP_ERR_CONFIG, "embedding: BVH traversal stack overflow");
  if (h[1] != ~0ull) throw StatusError(GMCP_ERR_DEGENERATE, "solve_barycentric_gram: near-degenerate edge basis");
}

void run_apply_embedding(Ctx& c, const int32_t* tri, const double* bary, const double* offset, int64_t n,
                         const int32_t* host_t, int64_t nht, const double* host_x, int64_t nhv, double* out,
                         int64_t* bad) {
  cudaStream_t s = c.stream;
  *bad = -1;
  if (n == 0) return;
  EmbedTmp& E = embed_tmp(c);
  E.tris.upload(host_t, 3 * nht, s);
  E.x.upload(host_x, 3 * nhv, s);
  E.tri.upload(tri, n, s);
  E.bary.upload(bary, 3 * n, s);
  E.off.upload(offset, n, s);
  E.out.resize(3 * n);
  E.bad.resize(3);
  GMCP_CUDA(cudaMemsetAsync(E.bad.p, 0xff, sizeof(unsigned long long), s));
  k_apply_embedding<<<grid_for(n, 256), 256, 0, s>>>(n, E.tri.p, E.bary.p, E.off.p, E.tris.p, E.x.p, E.out.p,
                                                      E.bad.p);
  ++c.launches;
  GMCP_CUDA(cudaGetLastError());
  unsigned long long h = 0;
  GMCP_CUDA(cudaMemcpyAsync(&h, E.bad.p, sizeof h, cudaMemcpyDeviceToHost, s));
  E.out.download(out, 3 * n, s);
  c.sync();
  if (h != ~0ull) {
    *bad = tri[h];
    throw StatusError(GMCP_ERR_DEGENERATE,
                      "host triangle " + std::to_string(tri[h]) + " is degenerate in the deformed configuration",
                      (int64_t)tri[h]);
  }
}

}  // namespace gmcp_b200

// CUB scan / sort / run-length helpers. Temp storage is the CubScratch of the
// context (or System) the current C-ABI call bound to this thread
// (common.cuh DeviceBind); all work on the caller's stream.
#pragma once

#include <cub/cub.cuh>

#include "common.cuh"

namespace gmcp_b200 {
namespace {

struct BoundScratch {
  void* get(size_t bytes) const {
    CubScratch* s = bound_scratch();
    if (!s) throw CudaError("gmcp_b200: CUB call outside a bound context");
    return s->get(bytes);
  }
};
constexpr BoundScratch g_scratch{};

template <class T>
void exclusive_scan(const T* in, T* out, int64_t n, cudaStream_t s) {
  size_t bytes = 0;
  GMCP_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n, s));
  void* t = g_scratch.get(bytes);
  GMCP_CUDA(cub::DeviceScan::ExclusiveSum(t, bytes, in, out, n, s));
}

// stable LSD radix sort (equal keys keep their input order)
template <class K, class V>
void sort_pairs(const K* kin, K* kout, const V* vin, V* vout, int64_t n, cudaStream_t s, int end_bit) {
  size_t bytes = 0;
  GMCP_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, bytes, kin, kout, vin, vout, n, 0, end_bit, s));
  void* t = g_scratch.get(bytes);
  GMCP_CUDA(cub::DeviceRadixSort::SortPairs(t, bytes, kin, kout, vin, vout, n, 0, end_bit, s));
}

template <class K>
void sort_keys(const K* kin, K* kout, int64_t n, cudaStream_t s, int end_bit) {
  size_t bytes = 0;
  GMCP_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, kin, kout, n, 0, end_bit, s));
  void* t = g_scratch.get(bytes);
  GMCP_CUDA(cub::DeviceRadixSort::SortKeys(t, bytes, kin, kout, n, 0, end_bit, s));
}

// unique keys of a sorted sequence with their counts; *num_out on the device
template <class K, class C>
void run_length_encode(const K* in, K* uniq, C* counts, C* num_out, int64_t n, cudaStream_t s) {
  size_t bytes = 0;
  GMCP_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, bytes, in, uniq, counts, num_out, n, s));
  void* t = g_scratch.get(bytes);
  GMCP_CUDA(cub::DeviceRunLengthEncode::Encode(t, bytes, in, uniq, counts, num_out, n, s));
}

}  // namespace
}  // namespace gmcp_b200

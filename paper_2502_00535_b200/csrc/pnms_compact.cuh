// pnms_compact.cuh — survivor masking (engine.py:284-293): scatter the sorted-order
// suppression bits back to input order, apply the implicit-padding gate, and compact the
// survivors into ascending input indices with a block-wide scan.
//
// Implicit padding: slots [count, d_max) are PADDING (0,0,0,0.0).  Row i then sees a padding
// column with z_j = 0, whose keep bit is always false (engine.py:232), so the row is
// suppressed iff gate(i, pad) holds, i.e. s_i < 0.0 (the by_index clause needs i > j, which
// never holds since i < count <= j).  NaN scores fail the comparison and survive.
#pragma once
#include "pnms_common.cuh"
#include "pnms_sort.cuh"

namespace pnms {

constexpr int kCompactThreads = 256;

struct CompactArgs {
  const double* s;
  const int32_t* counts;
  const int32_t* perm;
  const uint32_t* supp;
  const FrameMeta* meta;
  int batch, n_max, W32, d_max, tie_break;
  int32_t* keep_idx;       // may be null
  int32_t* keep_count;     // may be null
  uint32_t* keep_mask;     // may be null
  unsigned long long* gate_pairs;  // may be null
  const uint8_t* dense;   // optional [batch]: process frame f only if dense[f] != 0
  const int32_t* list;    // optional: process only frames list[0 .. *list_count) (grid-stride)
  const int* list_count;
};

__device__ __forceinline__ void compact_body(const CompactArgs& a, int f, unsigned char* smem_raw) {
  uint32_t* kbits = reinterpret_cast<uint32_t*>(smem_raw);          // [W32] survivor bits, input order
  uint32_t* warp_sums = kbits + ((a.W32 + 3) & ~3);
  const long long fbase = (long long)f * a.n_max;
  const int cnt = frame_count(a.counts, f, a.n_max);
  const int P = a.d_max > cnt ? a.d_max - cnt : 0;
  const uint32_t* supp_frame = a.supp + (long long)f * a.W32;

  for (int w = threadIdx.x; w < a.W32; w += kCompactThreads) kbits[w] = 0u;
  __syncthreads();
  // scatter sorted-order verdicts to input order (one shared atomic per survivor)
  for (int p = threadIdx.x; p < cnt; p += kCompactThreads) {
    const int i = a.perm[fbase + p];
    bool keep = !((supp_frame[p >> 5] >> (p & 31)) & 1u);
    if (P > 0 && keep && a.s[fbase + i] < 0.0) keep = false;
    if (keep) atomicOr(&kbits[i >> 5], 1u << (i & 31));
  }
  __syncthreads();

  const int words_per_thread = (a.W32 + kCompactThreads - 1) / kCompactThreads;
  const int w0 = threadIdx.x * words_per_thread;
  const int w1 = min(w0 + words_per_thread, a.W32);
  uint32_t local = 0;
  for (int w = w0; w < w1; ++w) {
    const uint32_t bits = kbits[w];
    local += __popc(bits);
    if (a.keep_mask) a.keep_mask[(long long)f * a.W32 + w] = bits;
  }
  uint32_t total;
  uint32_t pos = block_exclusive_scan(local, warp_sums, &total);
  if (a.keep_idx) {
    int32_t* out = a.keep_idx + fbase;
    for (int w = w0; w < w1; ++w) {
      uint32_t bits = kbits[w];
      while (bits) {
        out[pos++] = w * 32 + __ffs(bits) - 1;
        bits &= bits - 1;
      }
    }
  }
  if (threadIdx.x == 0) {
    if (a.keep_count) a.keep_count[f] = (int32_t)total;
    if (a.gate_pairs) {
      const FrameMeta fm = a.meta[f];
      const unsigned long long Pl = (unsigned long long)P;
      unsigned long long g = fm.lim_sum;
      g += Pl * (unsigned long long)fm.cnt_neg;                                  // (valid i, pad j)
      g += Pl * (unsigned long long)(fm.cnt_pos + (a.tie_break == 1 ? fm.cnt_zero : 0));  // (pad i, valid j)
      if (a.tie_break == 1 && P > 1) g += Pl * (Pl - 1) / 2;                     // (pad, pad)
      a.gate_pairs[f] = g;
    }
  }
}

__global__ void __launch_bounds__(kCompactThreads) pnms_compact(CompactArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  if (a.list) {
    // launched programmatically after the binned kernel (PDL): wait for its results
    pdl_wait();
    pdl_trigger();
    const int n = *a.list_count;
    for (int li = blockIdx.x; li < n; li += gridDim.x) {
      compact_body(a, a.list[li], smem_raw);
      __syncthreads();
    }
    return;
  }
  if (a.dense && !a.dense[blockIdx.x]) return;
  compact_body(a, blockIdx.x, smem_raw);
}

}  // namespace pnms

// pnms_small.cuh — single-launch latency path for calls with little total work (a single
// frame of up to a few thousand detections): the reference's own unsorted formulation
// (engine.py:204-244 + 253-281, Algorithm 1) — every ordered pair (i, j) is
// tested with the score gate evaluated per pair — spread over the whole GPU, with the
// survivor compaction (engine.py:284-293) done by the last CTA of each frame.
//
// Why unsorted here: a one-frame call cannot hide a sort behind other frames, and at
// n <= 4096 the doubled pair count costs less than the sort's serial latency.
//
// Work item = (frame, tile of 512 rows, tile of `cols` columns).  Columns are staged into
// shared memory; each thread owns four rows (one per 128-row group), so every column
// record read from shared memory serves four pair tests.  Per pair: the narrow7 overlap test of
// pnms_map.cuh plus the gate  sk_j < sk_i  (|| sk_j == sk_i && j < i  for by_index) on the
// 64-bit descending-order keys.  Verdicts are OR-ed into the frame's suppression words
// (input order).  Every CTA then takes a ticket; the frame's last CTA builds the survivor
// list and mask, adds the padding terms, and returns the frame's scratch words and counter
// to zero, so the workspace is clean for the next call without a memset.
#pragma once
#include "pnms_common.cuh"
#include "pnms_map.cuh"
#include "pnms_sort.cuh"

namespace pnms {

constexpr int kSmallThreads = 128;
constexpr int kSmallRowsMax = 4;       // rows per thread (1 for the tiniest calls, else 4)
// Persistent scratch at the start of every workspace (zero before the first call, left zero
// by every call): suppression words, per-frame tickets and gate accumulators.
constexpr int kSmallMaxWords = 4096;
constexpr int kSmallMaxFrames = 1024;
constexpr size_t kSmallScratchBytes = 128 * 1024;  // small path words + binned/tiles counters and masks
static_assert(kSmallMaxWords * 4 + kSmallMaxFrames * 4 + kSmallMaxFrames * 8 <= kSmallScratchBytes, "scratch");

struct SmallArgs {
  const int32_t *x, *y, *z;
  const double* s;
  const int32_t* counts;
  int batch, n_max, d_max, tie_break, W32;
  double theta;
  int cols, n_rt, n_ct;   // column tile width, row tiles and column tiles per frame
  uint32_t* supp;         // [batch][W32]  zero on entry and on exit
  unsigned int* ticket;   // [batch]       zero on entry and on exit
  unsigned long long* gacc;  // [batch]    zero on entry and on exit
  int32_t* keep_idx;
  int32_t* keep_count;
  uint32_t* keep_mask;
  unsigned long long* gate_pairs;
};

template <bool BY_INDEX, bool COUNT, int R>
__global__ void __launch_bounds__(kSmallThreads) pnms_small_kernel(SmallArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int s_wmode[kSmallThreads / 32];
  __shared__ unsigned int s_last;
  __shared__ unsigned long long s_gate;
  __shared__ uint32_t s_scan[kSmallThreads / 32 + 1];
  const int items = a.n_rt * a.n_ct;
  const int f = blockIdx.x / items;
  const int it = blockIdx.x % items;
  const int rt = it / a.n_ct, ct = it % a.n_ct;
  const long long fbase = (long long)f * a.n_max;
  const int cnt = frame_count(a.counts, f, a.n_max);
  const int r0 = rt * kSmallThreads * R, c0 = ct * a.cols;
  const int c1 = min(c0 + a.cols, cnt);
  const bool work = r0 < cnt && c0 < cnt;

  if (threadIdx.x == 0) s_gate = 0ull;
  // one global load phase: this thread's rows and (first) column into registers
  int32_t rx[R], ry[R], rz[R];
  double rs[R];
  int m = kNarrow7;
  if (work) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int i = r0 + r * kSmallThreads + threadIdx.x;
      rx[r] = ry[r] = rz[r] = 0;
      rs[r] = 0.0;
      if (i < cnt) {
        rx[r] = a.x[fbase + i]; ry[r] = a.y[fbase + i]; rz[r] = a.z[fbase + i]; rs[r] = a.s[fbase + i];
        m = max(m, frame_mode_of(rx[r], ry[r], rz[r]));
      }
    }
  }
  // the column tile in the same load phase: keys and narrow records straight into shared
  // memory (one global round trip); a tile that turns out not narrow7 rebuilds wide records
  uint64_t* ckey = reinterpret_cast<uint64_t*>(smem_raw);                       // [cols]
  uint8_t* crec = reinterpret_cast<uint8_t*>(ckey + a.cols);                     // [cols] records
  if (work) {
    for (int j = c0 + threadIdx.x; j < c1; j += kSmallThreads) {
      const long long g = fbase + j;
      const int32_t xv = a.x[g], yv = a.y[g], zv = a.z[g];
      m = max(m, frame_mode_of(xv, yv, zv));
      ckey[j - c0] = sort_key(a.s[g]);
      reinterpret_cast<RecNarrow*>(crec)[j - c0] = make_rec_narrow(xv, yv, zv, a.theta, kNarrow7);
    }
  }
  // the tile's arithmetic mode: one slot per warp (no shared initialisation to race with)
  m = __reduce_max_sync(0xFFFFFFFFu, m);
  if ((threadIdx.x & 31) == 0) s_wmode[threadIdx.x >> 5] = m;
  __syncthreads();
  int tile_mode = kNarrow7;
#pragma unroll
  for (int w = 0; w < kSmallThreads / 32; ++w) tile_mode = max(tile_mode, s_wmode[w]);
  // narrow16 tiles use the exact wide emulation (valid for every int32 input)
  const int mode = tile_mode == kNarrow7 ? kNarrow7 : kWide;
  if (work && mode == kWide) {
    for (int j = c0 + threadIdx.x; j < c1; j += kSmallThreads) {
      const long long g = fbase + j;
      reinterpret_cast<RecWide*>(crec)[j - c0] = make_rec_wide(a.x[g], a.y[g], a.z[g], a.theta);
    }
  }
  if (mode == kWide) __syncthreads();

  bool sup[R];
#pragma unroll
  for (int r = 0; r < R; ++r) sup[r] = false;
  if (work) {
    uint64_t ski[R];
    bool live[R];
    int idx[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      idx[r] = r0 + r * kSmallThreads + threadIdx.x;
      ski[r] = sort_key(rs[r]);
      live[r] = idx[r] < cnt && ski[r] != kNanSortKey;  // NaN rows never pass a gate
    }
    unsigned gcount = 0;
    if (mode == kWide) {
      const RecWide* cw = reinterpret_cast<const RecWide*>(crec);
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (!live[r]) continue;
        const RecWide ri = make_rec_wide(rx[r], ry[r], rz[r], a.theta);
        for (int j = c0; j < c1; ++j) {
          const uint64_t skj = ckey[j - c0];
          const bool gate = skj < ski[r] || (BY_INDEX && skj == ski[r] && j < idx[r]);
          if (COUNT) gcount += gate;
          if (gate && !sup[r]) sup[r] = suppress_wide(ri, cw[j - c0]);
        }
      }
    } else {
      uint32_t ra[R], rnb[R], rzz[R];
      int acc[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const RecNarrow rr = make_rec_narrow(rx[r], ry[r], rz[r], a.theta, kNarrow7);
        ra[r] = rr.a; rnb[r] = rr.nb; rzz[r] = rr.zz;
        acc[r] = -1;
        if (!live[r]) ski[r] = 0ull;  // no column key is below 0: the row never gates
      }
      const uint4* cn = reinterpret_cast<const uint4*>(crec);
#pragma unroll 4
      for (int j = c0; j < c1; ++j) {
        const uint64_t skj = ckey[j - c0];
        const uint4 cc = cn[j - c0];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const bool gate = skj < ski[r] || (BY_INDEX && skj == ski[r] && j < idx[r]);
          if (COUNT) gcount += gate;
          const int d = pair_d<kNarrow7>(ra[r], rnb[r], rzz[r], cc);
          acc[r] &= gate ? d : -1;
        }
      }
#pragma unroll
      for (int r = 0; r < R; ++r) sup[r] = live[r] && acc[r] >= 0;
    }
    if (COUNT) {
      const unsigned long long gw = __reduce_add_sync(0xFFFFFFFFu, gcount);
      if ((threadIdx.x & 31) == 0 && gw) atomicAdd(&s_gate, gw);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const uint32_t bits = __ballot_sync(0xFFFFFFFFu, sup[r]);
      if ((threadIdx.x & 31) == 0 && bits) atomicOr(a.supp + (long long)f * a.W32 + (idx[r] >> 5), bits);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (COUNT && s_gate) atomicAdd(a.gacc + f, s_gate);
    __threadfence();
    s_last = (atomicAdd(a.ticket + f, 1u) == (unsigned)(items - 1)) ? 1u : 0u;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();

  // ---- the frame's last CTA: survivor list, mask, counters; then clean the scratch
  const int P = a.d_max > cnt ? a.d_max - cnt : 0;
  uint32_t* supp_frame = a.supp + (long long)f * a.W32;
  const int wpt = (a.W32 + kSmallThreads - 1) / kSmallThreads;
  const int w0 = threadIdx.x * wpt, w1 = min(w0 + wpt, a.W32);
  uint32_t local = 0;
  for (int w = w0; w < w1; ++w) {
    const uint32_t sb = *((volatile uint32_t*)(supp_frame + w));
    const int base = w * 32;
    uint32_t valid = base + 32 <= cnt ? 0xFFFFFFFFu : (base >= cnt ? 0u : ((1u << (cnt - base)) - 1u));
    uint32_t keep = ~sb & valid;
    if (P > 0 && keep) {
      for (int t = 0; t < 32; ++t)
        if (((keep >> t) & 1u) && a.s[fbase + base + t] < 0.0) keep &= ~(1u << t);
    }
    local += __popc(keep);
    if (a.keep_mask) a.keep_mask[(long long)f * a.W32 + w] = keep;
  }
  uint32_t total;
  uint32_t pos = block_exclusive_scan(local, s_scan, &total);
  for (int w = w0; w < w1; ++w) {
    const uint32_t sb = *((volatile uint32_t*)(supp_frame + w));
    const int base = w * 32;
    uint32_t valid = base + 32 <= cnt ? 0xFFFFFFFFu : (base >= cnt ? 0u : ((1u << (cnt - base)) - 1u));
    uint32_t keep = ~sb & valid;
    if (P > 0 && keep) {
      for (int t = 0; t < 32; ++t)
        if (((keep >> t) & 1u) && a.s[fbase + base + t] < 0.0) keep &= ~(1u << t);
    }
    if (a.keep_idx) {
      while (keep) {
        a.keep_idx[fbase + pos++] = base + __ffs(keep) - 1;
        keep &= keep - 1;
      }
    }
  }
  __syncthreads();
  for (int w = threadIdx.x; w < a.W32; w += kSmallThreads) supp_frame[w] = 0u;
  if (COUNT) {
    // padding terms of map_writes (see pnms_compact.cuh)
    int neg = 0, pos_ = 0, zero = 0;
    for (int j = threadIdx.x; j < cnt; j += kSmallThreads) {
      const double v = a.s[fbase + j];
      neg += v < 0.0;
      pos_ += v > 0.0;
      zero += v == 0.0;
    }
    neg = __reduce_add_sync(0xFFFFFFFFu, neg);
    pos_ = __reduce_add_sync(0xFFFFFFFFu, pos_);
    zero = __reduce_add_sync(0xFFFFFFFFu, zero);
    __shared__ int s_cnt[3];
    if (threadIdx.x == 0) s_cnt[0] = s_cnt[1] = s_cnt[2] = 0;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) { atomicAdd(&s_cnt[0], neg); atomicAdd(&s_cnt[1], pos_); atomicAdd(&s_cnt[2], zero); }
    __syncthreads();
    if (threadIdx.x == 0 && a.gate_pairs) {
      const unsigned long long Pl = (unsigned long long)P;
      unsigned long long gp = *((volatile unsigned long long*)(a.gacc + f));
      gp += Pl * (unsigned long long)s_cnt[0];
      gp += Pl * (unsigned long long)(s_cnt[1] + (BY_INDEX ? s_cnt[2] : 0));
      if (BY_INDEX && P > 1) gp += Pl * (Pl - 1) / 2;
      a.gate_pairs[f] = gp;
    }
  }
  if (threadIdx.x == 0) {
    if (a.keep_count) a.keep_count[f] = (int32_t)total;
    if (COUNT) a.gacc[f] = 0ull;
    a.ticket[f] = 0u;
  }
}

}  // namespace pnms

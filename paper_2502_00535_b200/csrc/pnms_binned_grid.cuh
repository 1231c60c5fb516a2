// pnms_binned_grid.cuh — the exact binned NMS of pnms_binned.cuh for frames too large for one
// CTA's shared memory (> kBinMaxSlots slots, e.g. the 16384-box 4K frame of BASELINE config 3).
//
// One cooperative launch spans the whole GPU; frames are processed one after another, each in
// grid-synchronised phases over cell data kept in the workspace (L2-resident at these sizes):
//   stats -> cell histogram -> scan -> scatter in cell order -> candidate scan of the
//   reachable neighbour cells (per-pair score gate) -> compaction.
// Exactness argument and eligibility are those of pnms_binned.cuh; declined frames are
// flagged for the dense pipeline.
#pragma once
#include <cooperative_groups.h>

#include "pnms_binned.cuh"
#include "pnms_common.cuh"
#include "pnms_map.cuh"

namespace pnms {

namespace cg = cooperative_groups;

constexpr int kGridThreads = 512;
constexpr int kGridMaxCells = 1 << 16;

struct GridStats {
  int mode, minT, maxz, minx, miny, maxx, maxy, n_act, big, pad_[7];
};

struct BinGridArgs {
  const int32_t *x, *y, *z;
  const double* s;
  const int32_t* counts;
  int batch, n_max, d_max, tie_break, W32;
  double theta;
  // scratch (one frame at a time)
  RecNarrow* recS;     // [n_max]
  uint64_t* keyS;      // [n_max]
  int32_t* idxS;       // [n_max]
  int32_t* cellof;     // [n_max]
  uint32_t* cstart;    // [kGridMaxCells + 2]
  uint32_t* ccur;      // [kGridMaxCells + 2]
  uint32_t* kbits;     // [W32]
  GridStats* gst;
  uint8_t* fallback;   // [batch]
  int32_t* keep_idx;
  int32_t* keep_count;
  uint32_t* keep_mask;
};

inline size_t binned_grid_scratch_bytes(int n_max) {
  const size_t W32 = ((size_t)n_max + 31) / 32;
  return (size_t)n_max * (16 + 8 + 4 + 4) + (size_t)(kGridMaxCells + 4) * 4 * 2 + W32 * 4 + sizeof(GridStats) + 256;
}

template <bool BY_INDEX>
__global__ void __launch_bounds__(kGridThreads) pnms_binned_grid(BinGridArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ uint32_t scan_tmp[64];
  __shared__ uint32_t s_carry;
  const long long gtid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long gthreads = (long long)gridDim.x * blockDim.x;
  GridStats* st = a.gst;
  for (int f = 0; f < a.batch; ++f) {
    const long long fbase = (long long)f * a.n_max;
    const int cnt = frame_count(a.counts, f, a.n_max);
    if (gtid == 0) {
      st->mode = kNarrow7; st->minT = 0x7FFFFFFF; st->maxz = 0;
      st->minx = st->miny = 0x7FFFFFFF; st->maxx = st->maxy = -0x7FFFFFFF;
      st->n_act = 0; st->big = 0;
    }
    for (long long w = gtid; w < a.W32; w += gthreads) a.kbits[w] = 0u;
    for (long long c = gtid; c <= kGridMaxCells; c += gthreads) a.cstart[c] = 0u;
    grid.sync();
    // ---- statistics
    {
      int mode = kNarrow7, minT = 0x7FFFFFFF, maxz = 0, n_act = 0;
      int minx = 0x7FFFFFFF, miny = 0x7FFFFFFF, maxx = -0x7FFFFFFF, maxy = -0x7FFFFFFF;
      for (long long e = gtid; e < cnt; e += gthreads) {
        const long long g = fbase + e;
        const int32_t xv = a.x[g], yv = a.y[g], zv = a.z[g];
        const double sv = a.s[g];
        const int m = frame_mode_of(xv, yv, zv);
        mode = max(mode, m);
        if (sv == sv) {
          ++n_act;
          const int T = (m == kNarrow7) ? (int)((uint32_t)(-make_rec_narrow(xv, yv, zv, a.theta, kNarrow7).negT) >> 17) : 0;
          minT = min(minT, T);
          maxz = max(maxz, zv);
          minx = min(minx, xv); maxx = max(maxx, xv);
          miny = min(miny, yv); maxy = max(maxy, yv);
        }
      }
      mode = __reduce_max_sync(0xFFFFFFFFu, mode);
      minT = __reduce_min_sync(0xFFFFFFFFu, minT);
      maxz = __reduce_max_sync(0xFFFFFFFFu, maxz);
      n_act = __reduce_add_sync(0xFFFFFFFFu, n_act);
      minx = __reduce_min_sync(0xFFFFFFFFu, minx); maxx = __reduce_max_sync(0xFFFFFFFFu, maxx);
      miny = __reduce_min_sync(0xFFFFFFFFu, miny); maxy = __reduce_max_sync(0xFFFFFFFFu, maxy);
      if ((threadIdx.x & 31) == 0) {
        if (mode != kNarrow7) atomicMax(&st->mode, mode);
        atomicMin(&st->minT, minT); atomicMax(&st->maxz, maxz);
        if (n_act) atomicAdd(&st->n_act, n_act);
        atomicMin(&st->minx, minx); atomicMax(&st->maxx, maxx);
        atomicMin(&st->miny, miny); atomicMax(&st->maxy, maxy);
      }
    }
    grid.sync();
    const int n_act = *((volatile int*)&st->n_act);
    const bool eligible = *((volatile int*)&st->mode) == kNarrow7 && (n_act == 0 || *((volatile int*)&st->minT) >= 1);
    if (!eligible) {
      if (gtid == 0) a.fallback[f] = 1;
      grid.sync();
      continue;
    }
    const int maxz = *((volatile int*)&st->maxz);
    const int ox = *((volatile int*)&st->minx), oy = *((volatile int*)&st->miny);
    const int ex_ = *((volatile int*)&st->maxx), ey_ = *((volatile int*)&st->maxy);
    int S = maxz + 1, GX = 1, GY = 1;
    if (n_act > 0) {
      for (;;) {
        GX = (ex_ - ox) / S + 1;
        GY = (ey_ - oy) / S + 1;
        if ((long long)GX * GY <= kGridMaxCells) break;
        S *= 2;
      }
    }
    const int cells = GX * GY;
    // ---- cell histogram (NaN rows: survivors, no cell)
    for (long long e = gtid; e < cnt; e += gthreads) {
      const long long g = fbase + e;
      if (a.s[g] != a.s[g]) {
        atomicOr(&a.kbits[e >> 5], 1u << (e & 31));
        continue;
      }
      const int c = ((a.y[g] - oy) / S) * GX + (a.x[g] - ox) / S;
      a.cellof[e] = c;
      atomicAdd(&a.cstart[c], 1u);
    }
    grid.sync();
    // ---- exclusive scan of the cell counts (one CTA) + largest cell
    if (blockIdx.x == 0) {
      if (threadIdx.x == 0) s_carry = 0u;
      uint32_t big = 0;
      for (int base = 0; base < cells; base += kGridThreads) {
        const int c = base + threadIdx.x;
        const uint32_t v = c < cells ? a.cstart[c] : 0u;
        big = max(big, v);
        uint32_t total;
        const uint32_t ex = block_exclusive_scan(v, scan_tmp, &total);
        const uint32_t carry = s_carry;
        if (c < cells) { a.cstart[c] = carry + ex; a.ccur[c] = carry + ex; }
        __syncthreads();
        if (threadIdx.x == 0) s_carry = carry + total;
        __syncthreads();
      }
      big = __reduce_max_sync(0xFFFFFFFFu, big);
      if ((threadIdx.x & 31) == 0) atomicMax(&st->big, (int)big);
      if (threadIdx.x == 0) a.cstart[cells] = (uint32_t)n_act;
    }
    grid.sync();
    if (*((volatile int*)&st->big) > kBinCellMax) {
      if (gtid == 0) a.fallback[f] = 1;
      grid.sync();
      continue;
    }
    // ---- scatter into cell order
    for (long long e = gtid; e < cnt; e += gthreads) {
      const long long g = fbase + e;
      const double sv = a.s[g];
      if (sv != sv) continue;
      const uint32_t pos = atomicAdd(&a.ccur[a.cellof[e]], 1u);
      a.recS[pos] = make_rec_narrow(a.x[g], a.y[g], a.z[g], a.theta, kNarrow7);
      a.keyS[pos] = sort_key(sv);
      a.idxS[pos] = (int32_t)e;
    }
    grid.sync();
    // ---- candidate scan: every box of the reachable neighbour cells, with the per-pair gate
    // (cells are unordered here, so no early break on the gate; a found suppressor ends the row)
    const bool pad_rule = a.d_max > cnt;
    for (long long p = gtid; p < n_act; p += gthreads) {
      const int i = a.idxS[p];
      const uint64_t ki = a.keyS[p];
      const RecNarrow ri = a.recS[p];
      const int32_t ix = -(int32_t)(int16_t)(ri.nb & 0xFFFFu), iy = -(int32_t)(int16_t)(ri.nb >> 16);
      const int32_t iz = (int32_t)(ri.zz & 0xFFFFu) - 1;
      const int lx = ix - maxz - ox, ly = iy - maxz - oy;
      const int cx0 = lx < 0 ? 0 : lx / S, cy0 = ly < 0 ? 0 : ly / S;
      const int cx1 = min(GX - 1, (ix + iz - ox) / S), cy1 = min(GY - 1, (iy + iz - oy) / S);
      bool sup = false;
      for (int yy = cy0; yy <= cy1 && !sup; ++yy) {
        for (int xx = cx0; xx <= cx1 && !sup; ++xx) {
          const int c = yy * GX + xx;
          const int en = a.cstart[c + 1];
          for (int q = a.cstart[c]; q < en; ++q) {
            const uint64_t kj = a.keyS[q];
            const bool gate = kj < ki || (BY_INDEX && kj == ki && a.idxS[q] < i);
            const RecNarrow rj = a.recS[q];
            if (gate && pair_d<kNarrow7>(ri.a, ri.nb, ri.zz, make_uint4(rj.a, rj.nb, rj.zz, (uint32_t)rj.negT)) >= 0) {
              sup = true;
              break;
            }
          }
        }
      }
      if (!sup && pad_rule && a.s[fbase + i] < 0.0) sup = true;
      if (!sup) atomicOr(&a.kbits[i >> 5], 1u << (i & 31));
    }
    grid.sync();
    // ---- compaction (one CTA)
    if (blockIdx.x == 0) {
      if (threadIdx.x == 0) s_carry = 0u;
      __syncthreads();
      for (int base = 0; base < a.W32; base += kGridThreads) {
        const int w = base + threadIdx.x;
        const uint32_t bits = w < a.W32 ? *((volatile uint32_t*)&a.kbits[w]) : 0u;
        if (w < a.W32 && a.keep_mask) a.keep_mask[(long long)f * a.W32 + w] = bits;
        uint32_t total;
        uint32_t pos = block_exclusive_scan(__popc(bits), scan_tmp, &total) + s_carry;
        if (a.keep_idx) {
          uint32_t b = bits;
          while (b) {
            a.keep_idx[fbase + pos++] = w * 32 + __ffs(b) - 1;
            b &= b - 1;
          }
        }
        __syncthreads();
        if (threadIdx.x == 0) s_carry += total;
        __syncthreads();
      }
      if (threadIdx.x == 0) {
        if (a.keep_count) a.keep_count[f] = (int32_t)s_carry;
        a.fallback[f] = 0;
      }
    }
    grid.sync();
  }
}

}  // namespace pnms

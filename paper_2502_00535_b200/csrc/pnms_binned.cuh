// pnms_binned.cuh — exact spatially binned NMS, one CTA per frame, everything in shared
// memory.
//
// Exactness argument.  A pair with no pixel overlap has w*h = 0, and the reference
// suppresses on it only if 0 >= theta*(z_j+1)^2, i.e. only if T_j = 0 (theta = 0 or a
// zero-side slot, engine.py:229-232).  When every valid column has T_j >= 1, only pairs
// whose boxes overlap can suppress.  Boxes span [x, x+z] inclusive, so two overlapping boxes
// have |x_i - x_j| <= max side and |y_i - y_j| <= max side: with square cells of side
// S >= max_z + 1 their corner cells differ by at most one in each axis, and the 3x3
// neighbourhood of a box's cell holds every box that can suppress it.  Inside a cell the
// boxes are kept in (score desc, index asc) order, so the columns that pass the reference's
// gate (engine.py:233-235) form a prefix of each neighbour cell; the scan stops at the first
// column that fails the gate.  The result is the reference's row AND restricted to the only
// columns that can clear a bit — bit-identical survivors.
//
// Frames that do not meet the preconditions (a T_j = 0 column, coordinates outside the
// narrow7 domain, a cell holding more than kBinCellMax boxes, or > kBinMaxSlots slots) are
// flagged in `fallback[f]` and left to the dense sorted pipeline launched right after.
#pragma once
#include "pnms_common.cuh"
#include "pnms_map.cuh"
#include "pnms_sort.cuh"

namespace pnms {

constexpr int kBinThreads = 512;
constexpr int kBinMaxSlots = 4096;
constexpr int kBinMaxCells = 4096;   // upper bound; a frame uses at most max(64, npad) cells
constexpr int kBinCellMax = 64;

struct BinArgs {
  const int32_t *x, *y, *z;
  const double* s;
  const int32_t* counts;
  int batch, n_max, d_max, tie_break, W32;
  double theta;
  uint8_t* fallback;      // [batch] 1 = frame left to the dense pipeline
  int32_t* keep_idx;
  int32_t* keep_count;
  uint32_t* keep_mask;
  unsigned long long* pairs_tested;  // optional device counter (diagnostics), may be null
};

struct __align__(16) BinStats {
  int mode, minT, maxz, minx, miny, maxx, maxy, big, n_act, pad_;
};

__host__ __device__ inline int binned_max_cells(int npad) { return npad < 64 ? 64 : (npad > kBinMaxCells ? kBinMaxCells : npad); }
// npad is a multiple of 128, so every region below starts 16-byte aligned
__host__ __device__ inline int binned_npad(int n_max) { return (n_max + 127) & ~127; }
inline size_t binned_smem_bytes(int npad) {
  return (size_t)npad * (16 + 8 + 2 + 2) + (size_t)(binned_max_cells(npad) + 4) * 4 * 2 + (size_t)(npad / 32 + 4) * 4 +
         64 * 4 + sizeof(BinStats) + 64;
}

template <bool BY_INDEX>
__global__ void __launch_bounds__(kBinThreads) pnms_binned_frame(BinArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int f = blockIdx.x;
  const long long fbase = (long long)f * a.n_max;
  const int cnt = frame_count(a.counts, f, a.n_max);
  const int npad = binned_npad(a.n_max);
  // per-box data stored in cell order (positions [cstart[c], cstart[c+1]) = cell c)
  RecNarrow* recS = reinterpret_cast<RecNarrow*>(smem_raw);                   // [npad] records
  uint64_t* keyS = reinterpret_cast<uint64_t*>(recS + npad);                  // [npad] sort keys
  uint16_t* cellof = reinterpret_cast<uint16_t*>(keyS + npad);                // [npad] cell of input slot
  uint16_t* idxS = cellof + npad;                                             // [npad] input slot
  const int max_cells = binned_max_cells(npad);
  uint32_t* cstart = reinterpret_cast<uint32_t*>(idxS + npad);                // [cells+2]
  uint32_t* ccur = cstart + max_cells + 4;                                    // [cells+2]
  uint32_t* kbits = ccur + max_cells + 4;                                     // [npad/32] survivors
  uint32_t* scan_tmp = kbits + npad / 32 + 4;                                 // [64]
  BinStats* st = reinterpret_cast<BinStats*>(scan_tmp + 64);

  if (threadIdx.x == 0) {
    st->mode = kNarrow7; st->minT = 0x7FFFFFFF; st->maxz = 0;
    st->minx = st->miny = 0x7FFFFFFF; st->maxx = st->maxy = -0x7FFFFFFF;
    st->big = 0; st->n_act = 0;
  }
  for (int w = threadIdx.x; w < npad / 32; w += kBinThreads) kbits[w] = 0u;
  __syncthreads();
  if (a.n_max > kBinMaxSlots) {
    if (threadIdx.x == 0) a.fallback[f] = 1;
    return;
  }
  // ---- load: records, keys, frame statistics
  {
    int mode = kNarrow7, minT = 0x7FFFFFFF, maxz = 0, n_act = 0;
    int minx = 0x7FFFFFFF, miny = 0x7FFFFFFF, maxx = -0x7FFFFFFF, maxy = -0x7FFFFFFF;
    for (int e = threadIdx.x; e < cnt; e += kBinThreads) {
      const long long g = fbase + e;
      const int32_t xv = a.x[g], yv = a.y[g], zv = a.z[g];
      const uint64_t sk = sort_key(a.s[g]);
      const int m = frame_mode_of(xv, yv, zv);
      mode = max(mode, m);
      if (sk != kNanSortKey) {
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
      atomicMax(&st->mode, mode); atomicMin(&st->minT, minT); atomicMax(&st->maxz, maxz);
      atomicAdd(&st->n_act, n_act);
      atomicMin(&st->minx, minx); atomicMax(&st->maxx, maxx);
      atomicMin(&st->miny, miny); atomicMax(&st->maxy, maxy);
    }
  }
  __syncthreads();
  const bool eligible = st->mode == kNarrow7 && (st->n_act == 0 || st->minT >= 1);
  if (!eligible) {
    if (threadIdx.x == 0) a.fallback[f] = 1;
    return;
  }
  // ---- grid of square cells, side >= max side + 1
  int S = st->maxz + 1, GX = 1, GY = 1;
  if (st->n_act > 0) {
    for (;;) {
      GX = (st->maxx - st->minx) / S + 1;
      GY = (st->maxy - st->miny) / S + 1;
      if ((long long)GX * GY <= max_cells) break;
      S *= 2;
    }
  }
  const int cells = GX * GY, ox = st->minx, oy = st->miny;
  for (int c = threadIdx.x; c < cells + 1; c += kBinThreads) cstart[c] = 0u;
  __syncthreads();
  for (int e = threadIdx.x; e < cnt; e += kBinThreads) {
    if (a.s[fbase + e] != a.s[fbase + e]) {  // NaN: passes no gate, never suppresses -> survivor
      atomicOr(&kbits[e >> 5], 1u << (e & 31));
      continue;
    }
    const int32_t ex = a.x[fbase + e], ey = a.y[fbase + e];
    const int c = ((ey - oy) / S) * GX + (ex - ox) / S;
    cellof[e] = (uint16_t)c;
    atomicAdd(&cstart[c], 1u);
  }
  __syncthreads();
  // exclusive scan of the cell counts (+ largest cell)
  {
    const int per = (cells + 1 + kBinThreads - 1) / kBinThreads;
    const int b0 = threadIdx.x * per;
    uint32_t sum = 0, big = 0;
    for (int t = 0; t < per; ++t) {
      const int c = b0 + t;
      if (c < cells) { sum += cstart[c]; big = max(big, cstart[c]); }
    }
    big = __reduce_max_sync(0xFFFFFFFFu, big);
    if ((threadIdx.x & 31) == 0) atomicMax(&st->big, (int)big);
    uint32_t run = block_exclusive_scan(sum, scan_tmp, nullptr);
    for (int t = 0; t < per; ++t) {
      const int c = b0 + t;
      if (c < cells) { const uint32_t v = cstart[c]; cstart[c] = run; ccur[c] = run; run += v; }
    }
    if (threadIdx.x == 0) cstart[cells] = st->n_act;
  }
  __syncthreads();
  if (st->big > kBinCellMax) {
    if (threadIdx.x == 0) a.fallback[f] = 1;
    return;
  }
  // scatter records, keys and input slots straight into cell order
  for (int e = threadIdx.x; e < cnt; e += kBinThreads) {
    const long long g = fbase + e;
    const double sv = a.s[g];
    if (sv != sv) continue;
    const uint32_t pos = atomicAdd(&ccur[cellof[e]], 1u);
    recS[pos] = make_rec_narrow(a.x[g], a.y[g], a.z[g], a.theta, kNarrow7);
    keyS[pos] = sort_key(sv);
    idxS[pos] = (uint16_t)e;
  }
  __syncthreads();
  // ---- order every cell by (sort key asc == score desc, index asc): insertion sort
  for (int c = threadIdx.x; c < cells; c += kBinThreads) {
    const int b = cstart[c], en = cstart[c + 1];
    for (int i = b + 1; i < en; ++i) {
      const uint64_t kv = keyS[i];
      const uint16_t v = idxS[i];
      const RecNarrow rv = recS[i];
      int j = i - 1;
      while (j >= b) {
        const uint64_t ku = keyS[j];
        const uint16_t u = idxS[j];
        if (ku < kv || (ku == kv && u < v)) break;
        keyS[j + 1] = ku;
        idxS[j + 1] = u;
        recS[j + 1] = recS[j];
        --j;
      }
      keyS[j + 1] = kv;
      idxS[j + 1] = v;
      recS[j + 1] = rv;
    }
  }
  __syncthreads();
  // ---- scan: each valid box against the gate-passing prefix of its neighbour cells.  Rows
  // are taken in cell order so a warp's lanes walk the same few cell lists (broadcast reads,
  // similar trip counts).  A row only visits the cells its own extent can reach: a column j
  // overlapping row i has x_j in [x_i - max_z, x_i + z_i] (and the same for y).
  unsigned long long tested = 0;
  const int maxz = st->maxz;
  const bool pad_rule = a.d_max > cnt;
  for (int p = threadIdx.x; p < st->n_act; p += kBinThreads) {
    const int i = idxS[p];
    const uint64_t ki = keyS[p];
    const RecNarrow ri = recS[p];
    // corner and side back from the packed record: nb = (-x, -y), zz = (z+1, z+1)
    const int32_t ix = -(int32_t)(int16_t)(ri.nb & 0xFFFFu), iy = -(int32_t)(int16_t)(ri.nb >> 16);
    const int32_t iz = (int32_t)(ri.zz & 0xFFFFu) - 1;
    const int lx = ix - maxz - ox, ly = iy - maxz - oy;
    const int cx0 = lx < 0 ? 0 : lx / S, cy0 = ly < 0 ? 0 : ly / S;
    const int cx1 = min(GX - 1, (ix + iz - ox) / S), cy1 = min(GY - 1, (iy + iz - oy) / S);
    bool sup = false;
    for (int yy = cy0; yy <= cy1 && !sup; ++yy) {
      for (int xx = cx0; xx <= cx1 && !sup; ++xx) {
        const int c = yy * GX + xx;
        const int en = cstart[c + 1];
        for (int q = cstart[c]; q < en; ++q) {
          const uint64_t kj = keyS[q];
          const bool gate = kj < ki || (BY_INDEX && kj == ki && idxS[q] < i);
          if (!gate) break;
          ++tested;
          const RecNarrow rj = recS[q];
          if (pair_d<kNarrow7>(ri.a, ri.nb, ri.zz, make_uint4(rj.a, rj.nb, rj.zz, (uint32_t)rj.negT)) >= 0) {
            sup = true;
            break;
          }
        }
      }
    }
    // implicit padding gate (engine.py:233 with s_j = 0, z_j = 0): rows with s < 0 drop
    if (!sup && pad_rule && a.s[fbase + i] < 0.0) sup = true;
    if (!sup) atomicOr(&kbits[i >> 5], 1u << (i & 31));
  }
  if (a.pairs_tested) {
    tested = __reduce_add_sync(0xFFFFFFFFu, (unsigned)tested);
    if ((threadIdx.x & 31) == 0 && tested) atomicAdd(a.pairs_tested, tested);
  }
  __syncthreads();
  // ---- compaction (engine.py:284-293)
  const int words_per_thread = (a.W32 + kBinThreads - 1) / kBinThreads;
  const int w0 = threadIdx.x * words_per_thread, w1 = min(w0 + words_per_thread, a.W32);
  uint32_t local = 0;
  for (int w = w0; w < w1; ++w) {
    const uint32_t bits = kbits[w];
    local += __popc(bits);
    if (a.keep_mask) a.keep_mask[(long long)f * a.W32 + w] = bits;
  }
  uint32_t total;
  uint32_t pos = block_exclusive_scan(local, scan_tmp, &total);
  if (a.keep_idx) {
    for (int w = w0; w < w1; ++w) {
      uint32_t bits = kbits[w];
      while (bits) {
        a.keep_idx[fbase + pos++] = w * 32 + __ffs(bits) - 1;
        bits &= bits - 1;
      }
    }
  }
  if (threadIdx.x == 0) {
    if (a.keep_count) a.keep_count[f] = (int32_t)total;
    a.fallback[f] = 0;
  }
}

}  // namespace pnms

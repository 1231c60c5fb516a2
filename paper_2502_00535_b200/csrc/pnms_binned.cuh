// pnms_binned.cuh — exact spatially binned NMS, one CTA per frame, everything in shared
// memory.
//
// Exactness argument.  A pair with no pixel overlap has w*h = 0, and the reference
// suppresses on it only if 0 >= theta*(z_j+1)^2, i.e. only if T_j = 0 (theta = 0 or a
// zero-side slot, engine.py:229-232).  When every valid column has T_j >= 1, only pairs
// whose boxes overlap can suppress.  Boxes span [x, x+z] inclusive, so a column j that
// overlaps row i has its corner in [x_i - max_z, x_i + z_i] x [y_i - max_z, y_i + z_i]: with
// square cells of any side S, the cells that rectangle touches hold every box that can
// suppress row i (a 3x3 neighbourhood when S >= max_z + 1, more, smaller cells below).
// Inside a cell the boxes are kept in (score desc, index asc) order, so the columns that
// pass the reference's gate (engine.py:233-235) form a prefix of each cell; the scan stops
// at the first column that fails the gate.  The result is the reference's row AND
// restricted to the only columns that can clear a bit — bit-identical survivors.
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
constexpr int kBinMaxCells = 4096;   // upper bound; a frame uses at most max(64, 2 * npad) cells
constexpr int kBinCellMax = 255;  // skip (byte 1 of RecBin::w) and the 8-bit rank fields hold it

// Binned record (16 B, one LDS.128 per candidate column), narrow7 geometry as RecNarrow:
//   a  = (x+z+1, y+z+1), nb = (-x, -y)                       packed s16x2
//   w  = -(T << 17) | skip << 8 | (z+1)                       T = ceil(fl64(theta*(z+1)^2))
//   k  = high 32 bits of the 64-bit sort key (ascending == score descending)
// skip = boxes left to the end of the box's cell (<= kBinCellMax).  The pair value
// d = v*v + w = w_x^2 + skip*2^8 + (z+1) + (w_x*h - T)*2^17 keeps sign(w_x*h - T): the low
// terms stay below 16129 + 255*256 + 127 < 2^17 (the argument of pair_d).
// The full keys and input slots live in separate arrays: a suppressing column whose high key
// half equals the row's is verified on the full keys (rare: equal 32-bit prefixes).
struct __align__(16) RecBin {
  uint32_t a, nb;
  int32_t w;
  uint32_t k;
};
static_assert(sizeof(RecBin) == 16, "RecBin layout");

struct BinArgs {
  const int32_t *x, *y, *z;
  const double* s;
  const int32_t* counts;
  int batch, n_max, d_max, tie_break, W32;
  double theta;
  uint8_t* fallback;      // [batch] 1 = frame left to the dense pipeline
  int32_t* decl_list;     // declined frames, appended in any order ...
  int* decl_count;        // ... count (zero before the launch)
  FrameMeta* meta;        // optional: a declined frame's FrameMeta is zeroed (chunked dense path)
  int32_t* keep_idx;
  int32_t* keep_count;
  uint32_t* keep_mask;
  unsigned long long* pairs_tested;  // optional device counter (diagnostics), may be null
  unsigned long long* trace;         // optional per-CTA phase timestamps (diagnostics), may be null
  int cell_q8;                       // frame kernel cell side: 0 default, > 0 scale, < 0 absolute
  int cell_sx;                       // frame kernel: > 0 overrides the cell width
  int prefetch_ahead;                // frame kernel: > 0 prefetches frame f + this into L2
};

struct __align__(16) BinStats {
  int mode, minz, maxz, minx, miny, maxx, maxy, big, n_act, maxL, minW;  // (maxL/minW: tile kernel)
};

__host__ __device__ inline int binned_max_cells(int npad) {
  return npad < 32 ? 64 : (2 * npad > kBinMaxCells ? kBinMaxCells : 2 * npad);
}
// npad is a multiple of 128, so every region below starts 16-byte aligned
__host__ __device__ inline int binned_npad(int n_max) { return (n_max + 127) & ~127; }
inline size_t binned_smem_bytes(int npad) {
  return (size_t)npad * (sizeof(RecBin) + 8 + 2 + 2) + (size_t)(binned_max_cells(npad) + 4) * 4 +
         (size_t)(npad / 32 + 4) * 4 + 64 * 4 + sizeof(BinStats) + 64;
}
// boxes each thread keeps in registers between the load, binning and scatter passes
inline int binned_per_thread(int n_max, int threads) { return n_max <= 2 * threads ? 2 : (n_max <= 4 * threads ? 4 : 8); }

// floor(v / S) for 0 <= v < 2^16 as one IMAD.HI: M = floor(2^32 / S) + 1 is exact there
// (v * (M*S - 2^32) < 2^32) for 2 <= S < 2^15; S >= 2^15 makes every quotient 0 (M = 0).
// S = 1 has no 32-bit magic (2^32 + 1): callers keep every cell side >= 2 (kMinCellSide).
constexpr int kMinCellSide = 2;
__device__ __forceinline__ uint32_t div_magic(int S) {
  S = max(S, kMinCellSide);
  if (S >= 32768) return 0u;
  if ((S & (S - 1)) == 0) return 1u << (32 - (31 - __clz(S)));  // 2^32 / S: the same value, no division
  return (uint32_t)(0xFFFFFFFFu / (uint32_t)S) + 1u;
}
__device__ __forceinline__ int qdiv(int v, uint32_t M) { return (int)__umulhi((uint32_t)v, M); }

__device__ __forceinline__ void binned_decline(const BinArgs& a, int f) {
  a.fallback[f] = 1;
  if (a.meta) a.meta[f] = FrameMeta{};
  // the count starts at zero (workspace head); the bound keeps a workspace whose head was not
  // zeroed from writing past the list (the dispatcher clamps the count it reads)
  const int slot = atomicAdd(a.decl_count, 1);
  if (slot >= 0 && slot < a.batch) a.decl_list[slot] = f;
}

// diagnostics: global timer at phase boundaries of frame f (trace[f * 16 + phase]), thread 0;
// compiled into the COUNT (diagnostic) instantiations only — the checks cost ~3 % otherwise
#define PNMS_FRAME_TRACE(ph)                                                                   \
  do {                                                                                         \
    if (COUNT && a.trace && threadIdx.x == 0) {                                                \
      unsigned long long t_;                                                                   \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                   \
      a.trace[(long long)f * 16 + (ph)] = t_;                                                  \
    }                                                                                          \
  } while (0)

__device__ __forceinline__ uint4 lds128(uint32_t saddr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(saddr));
  return v;
}

// One row against one contiguous run of cells [qb, qe) (shared-window byte addresses of 16 B
// records in cell order; every cell in (key, slot) order, skip distance in bits 8..14 of w).
// Gate on the high key halves with <=: a superset of the reference's gate (engine.py:233-235)
// whose columns still form a prefix of every cell, so the scan jumps to the cell's end at the
// first column that fails it; a suppressor found with an equal half (or the row itself at pb)
// is verified on the full keys and slots outside the hot loop.  `base` is the address of
// record 0.  Returns true if the row is suppressed.
template <bool BY_INDEX, bool COUNT>
__device__ __forceinline__ bool binned_scan_run(uint32_t base, uint32_t qb, uint32_t qe, const RecBin& ri,
                                                uint32_t zzi, uint32_t pb, const uint64_t* keyS, const uint16_t* idxS,
                                                int p, unsigned long long& tested) {
  for (;;) {
    // branch-free body: the loop exits through its condition only (no break, so no
    // convergence-barrier bookkeeping per candidate)
    uint32_t gk = 0, step = 0;
    bool hit = false;
    bool go = qb < qe;
    while (go) {
      const uint4 g = lds128(qb);  // a, nb, w, k
      const bool gate = g.w <= ri.k;
      const uint32_t t1 = __viaddmin_s16x2(ri.a, g.y, zzi);
      const uint32_t t2 = __viaddmin_s16x2_relu(g.x, ri.nb, t1);
      const uint32_t v = __vimin_s16x2_relu(t2, __byte_perm(g.z, 0u, 0x4040));
      if (COUNT && gate) ++tested;
      hit = gate && (int)(v * v) + (int)g.z >= 0;
      gk = g.w;
      step = (gate ? 1u : __byte_perm(g.z, 0u, 0x4441)) << 4;
      qb += step;
      go = !hit && qb < qe;
    }
    if (!hit) return false;
    qb -= step;                   // back to the suppressor
    if (gk != ri.k) return true;  // strictly smaller high half: gated
    if (qb != pb) {               // equal halves: the reference's gate on the full key (and slot)
      const int q = (int)((qb - base) >> 4);
      const uint64_t kj = keyS[q], ki = keyS[p];
      if (kj < ki || (BY_INDEX && kj == ki && idxS[q] < idxS[p])) return true;
    }
    qb += (uint32_t)sizeof(RecBin);  // not gated (or the row itself): keep scanning
  }
}

// THREADS = 512 (three CTAs per SM: throughput) or 1024 (one CTA per SM, half the rows per
// thread: latency, for batches that fit one wave)
template <bool BY_INDEX, bool COUNT, int PER, int THREADS>
// returns true when the frame was declined (appended to the list for the dense pipeline)
__device__ __forceinline__ bool binned_frame_body(const BinArgs& a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int f = blockIdx.x;
  const long long fbase = (long long)f * a.n_max;
  const int cnt = frame_count(a.counts, f, a.n_max);
  const int npad = binned_npad(a.n_max);
  // the fallback kernels over the declined-frame list may launch once every CTA has started
  // (programmatic dependent launch); they wait for this grid's completion before reading
  pdl_trigger();
  PNMS_FRAME_TRACE(0);
  // per-box data stored in cell order (positions [cstart[c], cstart[c+1]) = cell c)
  RecBin* recS = reinterpret_cast<RecBin*>(smem_raw);                         // [npad] records
  uint64_t* keyS = reinterpret_cast<uint64_t*>(recS + npad);                  // [npad] full sort keys
  uint16_t* idxS = reinterpret_cast<uint16_t*>(keyS + npad);                  // [npad] input slots
  const int max_cells = binned_max_cells(npad);
  uint32_t* cstart = reinterpret_cast<uint32_t*>(idxS + npad);                // [cells+2]
  uint32_t* kbits = cstart + max_cells + 4;                                   // [npad/32] survivors
  uint32_t* scan_tmp = kbits + npad / 32 + 4;                                 // [64]
  BinStats* st = reinterpret_cast<BinStats*>(scan_tmp + 64);
  uint16_t* cpos = reinterpret_cast<uint16_t*>(st + 1);  // [npad] cell, then rank, of arrival position p

  if (threadIdx.x == 0) {
    st->mode = kNarrow7; st->minz = 0x7FFFFFFF; st->maxz = 0;
    st->minx = st->miny = 0x7FFFFFFF; st->maxx = st->maxy = -0x7FFFFFFF;
    st->big = 0; st->n_act = 0;
  }
  for (int w = threadIdx.x; w < npad / 32; w += THREADS) kbits[w] = 0u;
  __syncthreads();
  if (a.n_max > PER * THREADS) {
    if (threadIdx.x == 0) binned_decline(a, f);
    return true;
  }
  // ---- pass 1: the frame is read from HBM once; each thread keeps its PER boxes in
  // registers (xy packed as two 16-bit halves — exact for every frame that stays on this
  // path — and z | cell << 16 | rank-in-cell << 8 later).  Frame statistics.
  uint32_t xy[PER], zc[PER];
  {
    int mode = kNarrow7, minz = 0x7FFFFFFF, maxz = 0, n_act = 0;
    int minx = 0x7FFFFFFF, miny = 0x7FFFFFFF, maxx = -0x7FFFFFFF, maxy = -0x7FFFFFFF;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int e = threadIdx.x + k * THREADS;
      xy[k] = 0u; zc[k] = 0xFFFFFFFFu;  // 0xFFFFFFFF = no box (slot >= count, or NaN score)
      if (e < cnt) {
        const long long g = fbase + e;
        const int32_t xv = a.x[g], yv = a.y[g], zv = a.z[g];
        const double sv = a.s[g];
        mode = max(mode, frame_mode_of(xv, yv, zv));
        if (sv == sv) {
          ++n_act;
          minz = min(minz, zv); maxz = max(maxz, zv);
          minx = min(minx, xv); maxx = max(maxx, xv);
          miny = min(miny, yv); maxy = max(maxy, yv);
          xy[k] = ((uint32_t)xv & 0xFFFFu) | ((uint32_t)yv << 16);
          zc[k] = (uint32_t)zv & 0xFFu;
        } else {
          atomicOr(&kbits[e >> 5], 1u << (e & 31));  // NaN: passes no gate, never suppresses -> survivor
        }
      }
    }
    mode = __reduce_max_sync(0xFFFFFFFFu, mode);
    minz = __reduce_min_sync(0xFFFFFFFFu, minz);
    maxz = __reduce_max_sync(0xFFFFFFFFu, maxz);
    n_act = __reduce_add_sync(0xFFFFFFFFu, n_act);
    minx = __reduce_min_sync(0xFFFFFFFFu, minx); maxx = __reduce_max_sync(0xFFFFFFFFu, maxx);
    miny = __reduce_min_sync(0xFFFFFFFFu, miny); maxy = __reduce_max_sync(0xFFFFFFFFu, maxy);
    if ((threadIdx.x & 31) == 0) {
      atomicMax(&st->mode, mode); atomicMin(&st->minz, minz); atomicMax(&st->maxz, maxz);
      atomicAdd(&st->n_act, n_act);
      atomicMin(&st->minx, minx); atomicMax(&st->maxx, maxx);
      atomicMin(&st->miny, miny); atomicMax(&st->maxy, maxy);
    }
  }
  __syncthreads();
  PNMS_FRAME_TRACE(1);
  // T_j >= 1 for every active column  <=>  theta > 0 and no zero side (T = 0 only for z = 0,
  // engine.py:232, or theta*(z+1)^2 == 0)
  const int n_act = st->n_act;
  const bool eligible = st->mode == kNarrow7 && (n_act == 0 || (a.theta > 0.0 && st->minz >= 1));
  if (!eligible) {
    if (threadIdx.x == 0) binned_decline(a, f);
    return true;
  }
  // ---- grid of cells, Sx wide and Sy tall.  Any sides are exact (a column that can suppress
  // row i has its corner in [x_i - max_z, x_i + z_i] x [y_i - max_z, y_i + z_i]).  A row scans
  // one contiguous run of cells per cell row it reaches, so narrow cells tighten the x range at
  // no cost in runs while tall cells cut the runs per row.  Default: Sy = the power of two
  // nearest max_z + 1, Sx = Sy / 4 — measured on BASELINE config 5 (max_z = 64, 2048 boxes of
  // 1920x1080): 16 x 64 cells 0.65 ms, 12 x 64 0.645, 24 x 64 0.66, 16 x 48 0.70, 16 x 80 0.74,
  // 32 x 32 0.68, 65 x 65 (3x3 neighbourhoods) 0.76 (tools/env_sweep.py PNMS_CELL_SX ...).
  // Tuning: cell_q8 < 0 sets square cells of side -cell_q8, > 0 scales (max_z + 1) by
  // cell_q8 / 256 for both; cell_sx > 0 then overrides the width.
  int Sx, Sy;
  if (a.cell_q8 == 0) {
    const int h = st->maxz + 1;
    const int p2 = 1 << (31 - __clz(h));
    Sy = (long long)h * h > 2LL * p2 * p2 ? 2 * p2 : p2;
    Sx = Sy >> 2;
  } else {
    Sy = a.cell_q8 < 0 ? -a.cell_q8 : ((st->maxz + 1) * a.cell_q8 + 255) >> 8;
    Sx = Sy;
  }
  if (a.cell_sx > 0) Sx = a.cell_sx;
  Sx = max(Sx, kMinCellSide);  // div_magic needs sides >= 2
  Sy = max(Sy, kMinCellSide);
  int GX = 1, GY = 1;
  const int ox = st->minx, oy = st->miny;
  if (n_act > 0) {
    for (;;) {
      GX = (st->maxx - ox) / Sx + 1;
      GY = (st->maxy - oy) / Sy + 1;
      if ((long long)GX * GY <= max_cells) break;
      if (Sx < Sy) Sx *= 2;  // too many cells: widen first, then grow both
      else { Sx *= 2; Sy *= 2; }
    }
  }
  const uint32_t Mx = div_magic(Sx), My = div_magic(Sy);
  const int cells = GX * GY;
  for (int c = threadIdx.x; c < cells + 1; c += THREADS) cstart[c] = 0u;
  __syncthreads();
  PNMS_FRAME_TRACE(2);
  // ---- pass 2: histogram; the atomic's return value is the box's rank inside its cell
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    if (zc[k] != 0xFFFFFFFFu) {
      const int ex = (int)(xy[k] & 0xFFFFu), ey = (int)(xy[k] >> 16);
      const int c = qdiv(ey - oy, My) * GX + qdiv(ex - ox, Mx);
      const uint32_t r = atomicAdd(&cstart[c], 1u);
      zc[k] |= ((uint32_t)c << 16) | (min(r, 255u) << 8);
    }
  }
  __syncthreads();
  PNMS_FRAME_TRACE(3);
  // exclusive scan of the cell counts (+ largest cell)
  {
    const int per = (cells + 1 + THREADS - 1) / THREADS;
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
      if (c < cells) { const uint32_t v = cstart[c]; cstart[c] = run; run += v; }
    }
    if (threadIdx.x == 0) cstart[cells] = n_act;
  }
  __syncthreads();
  PNMS_FRAME_TRACE(4);
  if (st->big > kBinCellMax) {
    if (threadIdx.x == 0) binned_decline(a, f);
    return true;
  }
  // ---- pass 3: keys, slots and cells into cell order by arrival; then one thread per arrival
  // position counts the members of its cell that precede it in (key, slot) order — a parallel
  // rank sort whose adjacent lanes share a cell (uniform trip counts) — and after a barrier
  // every box writes its record, key and slot at the final position with the distance to its
  // cell's end
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    if (zc[k] != 0xFFFFFFFFu) {
      const int e = threadIdx.x + k * THREADS;
      const uint32_t pos = cstart[zc[k] >> 16] + ((zc[k] >> 8) & 0xFFu);
      keyS[pos] = sort_key(a.s[fbase + e]);
      idxS[pos] = (uint16_t)e;
      cpos[pos] = (uint16_t)(zc[k] >> 16);
    }
  }
  __syncthreads();
  PNMS_FRAME_TRACE(5);
  {
    // high key halves (one 32-bit load per member); members with an equal half other than the
    // box itself are rare and resolved exactly in a second loop
    const uint32_t* khi = reinterpret_cast<const uint32_t*>(keyS) + 1;
    for (int p = threadIdx.x; p < n_act; p += THREADS) {
      const int c = cpos[p];
      const int b = (int)cstart[c], en = (int)cstart[c + 1];
      const uint32_t hi = khi[2 * p];
      int rank = 0, eq = 0;
      for (int j = b; j < en; ++j) {
        const uint32_t hj = khi[2 * j];
        rank += hj < hi;
        eq += hj == hi;
      }
      if (eq > 1) {
        const uint64_t key = keyS[p];
        const int e = idxS[p];
        rank = 0;
        for (int j = b; j < en; ++j) {
          const uint64_t kj = keyS[j];
          rank += kj < key || (kj == key && (int)idxS[j] < e);
        }
      }
      cpos[p] = (uint16_t)rank;  // own slot; < kBinCellMax
    }
  }
  __syncthreads();
  PNMS_FRAME_TRACE(6);
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    if (zc[k] != 0xFFFFFFFFu) {
      const int e = threadIdx.x + k * THREADS;
      const int c = (int)(zc[k] >> 16);
      const int b = (int)cstart[c];
      const int pos = b + (int)cpos[b + ((zc[k] >> 8) & 0xFFu)];
      const int en = (int)cstart[c + 1];
      const int32_t xv = (int32_t)(xy[k] & 0xFFFFu), yv = (int32_t)(xy[k] >> 16), zv = (int32_t)(zc[k] & 0xFFu);
      const RecNarrow rn = make_rec_narrow(xv, yv, zv, a.theta, kNarrow7);
      const uint64_t key = sort_key(a.s[fbase + e]);
      RecBin rb;
      rb.a = rn.a; rb.nb = rn.nb; rb.w = rn.negT | (zv + 1) | ((en - pos) << 8); rb.k = (uint32_t)(key >> 32);
      recS[pos] = rb;
      keyS[pos] = key;
      idxS[pos] = (uint16_t)e;
    }
  }
  __syncthreads();
  PNMS_FRAME_TRACE(7);
  // ---- scan: each valid box against the gate-passing prefix of every cell its extent can
  // reach.  A column j overlapping row i has x_j in [x_i - max_z, x_i + z_i] (same for y), so
  // the reachable cells of one cell row are contiguous in cell order: one run per cell row.
  // Inside a run the scan jumps to the end of the current cell at the first column that
  // fails the gate (the cell's gate-passing columns are its prefix).
  unsigned long long tested = 0;
  const int maxz = st->maxz;
  const bool pad_rule = a.d_max > cnt;
  const uint32_t rbase = static_cast<uint32_t>(__cvta_generic_to_shared(recS));
  for (int p = threadIdx.x; p < n_act; p += THREADS) {
    const RecBin ri = recS[p];
    const uint32_t zzi = __byte_perm((uint32_t)ri.w, 0u, 0x4040);  // (z+1, z+1)
    // corner and side back from the packed record: nb = (-x, -y)
    const int32_t ix = -(int32_t)(int16_t)(ri.nb & 0xFFFFu), iy = -(int32_t)(int16_t)(ri.nb >> 16);
    const int32_t iz = (int32_t)(ri.w & 0xFF) - 1;
    const int cx0 = qdiv(max(ix - maxz - ox, 0), Mx), cy0 = qdiv(max(iy - maxz - oy, 0), My);
    const int cx1 = min(GX - 1, qdiv(ix + iz - ox, Mx)), cy1 = min(GY - 1, qdiv(iy + iz - oy, My));
    const uint32_t pb = rbase + (uint32_t)p * (uint32_t)sizeof(RecBin);
    bool sup = false;
    for (int yy = cy0; yy <= cy1 && !sup; ++yy) {
      // byte offsets of the run's first record and its end
      const uint32_t qb = rbase + cstart[yy * GX + cx0] * (uint32_t)sizeof(RecBin);
      const uint32_t qe = rbase + cstart[yy * GX + cx1 + 1] * (uint32_t)sizeof(RecBin);
      if (binned_scan_run<BY_INDEX, COUNT>(rbase, qb, qe, ri, zzi, pb, keyS, idxS, p, tested)) sup = true;
    }
    const int i = idxS[p];
    // implicit padding gate (engine.py:233 with s_j = 0, z_j = 0): rows with s < 0 drop
    if (!sup && pad_rule && a.s[fbase + i] < 0.0) sup = true;
    if (!sup) atomicOr(&kbits[i >> 5], 1u << (i & 31));
  }
  if (COUNT && a.pairs_tested) {
    tested = __reduce_add_sync(0xFFFFFFFFu, (unsigned)tested);
    if ((threadIdx.x & 31) == 0 && tested) atomicAdd(a.pairs_tested, tested);
  }
  __syncthreads();
  PNMS_FRAME_TRACE(8);
  // ---- compaction (engine.py:284-293)
  const int words_per_thread = (a.W32 + THREADS - 1) / THREADS;
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
  PNMS_FRAME_TRACE(9);
  return false;
}

template <bool BY_INDEX, bool COUNT, int PER, int THREADS>
__global__ void __launch_bounds__(THREADS, (THREADS == 512 ? 3 : 1)) pnms_binned_frame(BinArgs a) {
  binned_frame_body<BY_INDEX, COUNT, PER, THREADS>(a);
}

}  // namespace pnms

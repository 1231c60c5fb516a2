// pnms_binned2.cuh — exact spatially binned NMS, one CTA per frame, with exact score ranks,
// a theta-tightened reach and rows scanned in order of their candidate counts.
//
// Same contract and exactness argument as pnms_binned.cuh (the reference's row AND of
// engine.py:204-281 restricted to the only columns that can clear a bit), with three changes
// that cut the kernel's instruction count (it is issue-bound):
//
//  1. Reach from theta.  A column j clears bit (i,j) only if w*h >= T_j with
//     T_j = ceil(fl64(theta*(z_j+1)^2)) (engine.py:229-232).  Both extents are at most z_j+1,
//     so each one is at least wmin_j = ceil(T_j / (z_j+1)).  With w <= x_j+z_j-x_i+1 and
//     w <= x_i+z_i-x_j+1 every such column has
//         x_j in [x_i - L, x_i + z_i + 1 - R],   L = max_j (z_j + 1 - wmin_j),  R = min_j wmin_j
//     (same for y), L and R taken over the frame's active boxes.  At theta = 0.5 that is about
//     half of max_z to the left and R ~ min_z/2 less to the right: ~2.4x fewer candidates than
//     the [x_i - max_z, x_i + z_i] window of pnms_binned.cuh.
//  2. Exact 32-bit ranks instead of in-cell key order.  Every active box gets its rank in
//     (score desc[, index asc for by_index]) order from a value-linear bucket sort of the
//     high key halves with an exact in-bucket count on the full 64-bit keys.  The gate of
//     engine.py:233-235 becomes rank_j < rank_i (equal scores share a rank under
//     paper_faithful and never gate each other; the row itself never passes), so the scan has
//     no verification path and the cells need no internal order: records are written once.
//  3. Balanced rows.  Each row's candidates (every record in the cells of its window, one
//     contiguous run per cell row) are counted when its record is written; rows are then
//     scanned in ascending order of that count, so the 32 lanes of a warp walk runs of
//     similar length.  A lane walks all runs of its row in one flattened loop (item k maps to
//     its run through three compares), exiting at the first suppressor.
//
// Declined (left to the dense pipeline through the device-side list, as pnms_binned.cuh):
// frames outside narrow7, with a T_j = 0 column (theta = 0 or a zero side), more than
// PER*THREADS slots, or a tie group larger than kB2BucketMax (in-bucket counting is quadratic).
#pragma once
#include "pnms_binned.cuh"

namespace pnms {

constexpr int kB2RowClasses = 64;   // rows are ordered by min(candidates, 63)
constexpr int kB2RunGroup = 4;      // runs a row walks in one flattened loop
constexpr int kB2BucketMax = 512;   // largest score bucket counted in place

struct __align__(16) B2Stats {
  // per-frame statistics (shared atomics)
  int mode, minz, maxz, minx, miny, maxx, maxy, n_act;
  int maxL, minW, done, big;
  uint32_t fmin, fmax;  // order-preserving bits of the finite fp32 scores
  // derived by the last warp to finish the statistics
  int eligible, L, R, GX, GY, cells, ox, oy;
  uint32_t Mx, My;
  float smin, inv;
};

// Compile-time shared-memory layout for NP = PER * THREADS slots: records, bucket-order keys
// (later the row order), cell-order and bucket-order input slots, the u16 counters
// [cells | buckets | 0], survivor bits, the T table, the row-class histogram, scan scratch.
template <int NP>
struct B2Layout {
  static constexpr int kMaxCells = 2 * NP;
  static constexpr int kBuckets = 2 * NP;  // a power of two
  static constexpr int kComb = kMaxCells + kBuckets + 8;  // + sentinel, in whole uint4
  static constexpr size_t oRec = 0;
  static constexpr size_t oKey = oRec + 16 * (size_t)NP;
  static constexpr size_t oIdxS = oKey + 8 * (size_t)NP;
  static constexpr size_t oIdxB = oIdxS + 2 * (size_t)NP;
  static constexpr size_t oComb = oIdxB + 2 * (size_t)NP;
  static constexpr size_t oBits = oComb + 2 * (size_t)kComb;
  static constexpr size_t oTz = oBits + 4 * (size_t)(NP / 32);
  static constexpr size_t oHist = oTz + 4 * 128;
  static constexpr size_t oScan = oHist + 4 * kB2RowClasses;
  static constexpr size_t oSt = oScan + 4 * 64;
  static constexpr size_t kBytes = oSt + sizeof(B2Stats);
  static_assert(NP % 256 == 0, "NP: a multiple of 256");
  static_assert(oComb % 16 == 0 && oBits % 16 == 0 && oSt % 16 == 0, "alignment");
};
inline size_t b2_smem_bytes(int np) {
  return np <= 1024 ? B2Layout<1024>::kBytes : (np <= 2048 ? B2Layout<2048>::kBytes : B2Layout<4096>::kBytes);
}

// 16-bit counter increment through the u32 word holding it; returns the old count (counts
// stay below 2^16, so the low half never carries into the high half)
__device__ __forceinline__ uint32_t atomic_inc_u16(uint16_t* base, int idx) {
  uint32_t* w = reinterpret_cast<uint32_t*>(base) + (idx >> 1);
  const int sh = (idx & 1) << 4;
  return (atomicAdd(w, 1u << sh) >> sh) & 0xFFFFu;
}
// order-preserving u32 of a float (and back)
__device__ __forceinline__ uint32_t f32_key(float v) {
  const uint32_t b = __float_as_uint(v);
  return (b >> 31) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float f32_unkey(uint32_t k) { return __uint_as_float((k >> 31) ? (k & 0x7FFFFFFFu) : ~k); }

template <bool BY_INDEX, bool COUNT, int PER, int THREADS>
__device__ __forceinline__ bool binned2_frame_body(const BinArgs& a) {
  constexpr int NP = PER * THREADS;
  using Ly = B2Layout<NP>;
  constexpr int NW = THREADS / 32;
  constexpr int NB = Ly::kBuckets;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int f = blockIdx.x;
  const long long fbase = (long long)f * a.n_max;
  const int cnt = frame_count(a.counts, f, a.n_max);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  pdl_trigger();
  PNMS_FRAME_TRACE(0);
  if (a.prefetch_ahead > 0 && threadIdx.x < 4 && f + a.prefetch_ahead < a.batch) {
    // the frame that will run on this CTA slot next: its planes into L2 while this one runs
    const long long pf = (long long)(f + a.prefetch_ahead) * a.n_max;
    const void* src = threadIdx.x == 0 ? (const void*)(a.x + pf) : threadIdx.x == 1 ? (const void*)(a.y + pf)
                    : threadIdx.x == 2 ? (const void*)(a.z + pf) : (const void*)(a.s + pf);
    const uint32_t bytes = (uint32_t)a.n_max * (threadIdx.x == 3 ? 8u : 4u);
    if ((reinterpret_cast<uintptr_t>(src) & 15) == 0)
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes & ~15u) : "memory");
  }
  RecBin* recS = reinterpret_cast<RecBin*>(smem_raw + Ly::oRec);        // records, cell order
  uint64_t* keyB = reinterpret_cast<uint64_t*>(smem_raw + Ly::oKey);    // keys, bucket order
  uint16_t* order = reinterpret_cast<uint16_t*>(smem_raw + Ly::oKey);   //   later: rows by count
  uint16_t* idxS = reinterpret_cast<uint16_t*>(smem_raw + Ly::oIdxS);   // input slot, cell order
  uint16_t* idxB = reinterpret_cast<uint16_t*>(smem_raw + Ly::oIdxB);   // input slot, bucket order
  uint16_t* comb = reinterpret_cast<uint16_t*>(smem_raw + Ly::oComb);   // cell | bucket counts | 0
  uint32_t* kbits = reinterpret_cast<uint32_t*>(smem_raw + Ly::oBits);  // survivors, input order
  uint32_t* Tz = reinterpret_cast<uint32_t*>(smem_raw + Ly::oTz);       // T | wmin << 16
  uint32_t* rowhist = reinterpret_cast<uint32_t*>(smem_raw + Ly::oHist);
  uint32_t* scan_tmp = reinterpret_cast<uint32_t*>(smem_raw + Ly::oScan);
  B2Stats* st = reinterpret_cast<B2Stats*>(smem_raw + Ly::oSt);

  // the frame's loads are issued first, so their latency overlaps the initialisation below
  // and its barrier (the n_max > NP case declines before using them)
  int32_t lx[PER], ly[PER], lz[PER];
  double ls[PER];
  if (a.n_max <= NP) {
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int e = threadIdx.x + k * THREADS;
      const long long g = fbase + (e < cnt ? e : 0);
      lx[k] = e < cnt ? a.x[g] : 0; ly[k] = e < cnt ? a.y[g] : 0; lz[k] = e < cnt ? a.z[g] : 0;
      ls[k] = e < cnt ? a.s[g] : 0.0;
    }
  }
  if (threadIdx.x == 0) {
    st->mode = kNarrow7; st->minz = 0x7FFFFFFF; st->maxz = 0;
    st->minx = st->miny = 0x7FFFFFFF; st->maxx = st->maxy = -0x7FFFFFFF;
    st->n_act = 0; st->maxL = 0; st->minW = 0x7FFFFFFF; st->done = 0; st->big = 0;
    st->fmin = 0xFFFFFFFFu; st->fmax = 0u;
  }
  for (int w = threadIdx.x; w < Ly::kComb / 8; w += THREADS)
    reinterpret_cast<uint4*>(comb)[w] = make_uint4(0u, 0u, 0u, 0u);
  if (threadIdx.x < kB2RowClasses) rowhist[threadIdx.x] = 0u;
  if (threadIdx.x < 128) {
    // T_z = ceil(fl64(theta*(z+1)^2)) (engine.py:197, 229-232; 0 for z = 0) and the least
    // extent a suppressing column of side z needs, wmin_z = ceil(T_z / (z+1))
    const int zv = threadIdx.x;
    const uint32_t T = zv == 0 ? 0u : (uint32_t)ceil(ref_threshold(a.theta, zv));
    Tz[zv] = T | (((T + zv) / (uint32_t)(zv + 1)) << 16);
  }
  __syncthreads();
  if (a.n_max > NP) {
    if (threadIdx.x == 0) binned_decline(a, f);
    return true;
  }
  const bool pad_rule = a.d_max > cnt;
  // ---- pass 1: the frame is read from HBM once into registers; statistics; survivor bits
  // start set for every valid slot except rows the padding columns suppress (engine.py:233 with
  // s_j = 0, z_j = 0: s_i < 0), NaN rows included (they pass no gate and never suppress)
  uint32_t xy[PER], zc[PER], bb[PER];
  uint64_t* keyIn = reinterpret_cast<uint64_t*>(recS);  // keys by input slot until the records
  {
    int mode = kNarrow7, minz = 0x7FFFFFFF, maxz = 0, n_act = 0, maxL = 0, minW = 0x7FFFFFFF;
    int minx = 0x7FFFFFFF, miny = 0x7FFFFFFF, maxx = -0x7FFFFFFF, maxy = -0x7FFFFFFF;
    uint32_t fmin = 0xFFFFFFFFu, fmax = 0u;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int e = threadIdx.x + k * THREADS;
      xy[k] = 0u; zc[k] = 0xFFFFFFFFu; bb[k] = 0u;
      bool keep = false;
      if (e < cnt) {
        const int32_t xv = lx[k], yv = ly[k], zv = lz[k];
        const double sv = ls[k];
        mode = max(mode, frame_mode_of(xv, yv, zv));
        keep = !(pad_rule && sv < 0.0);
        if (sv == sv) {
          ++n_act;
          minz = min(minz, zv); maxz = max(maxz, zv);
          minx = min(minx, xv); maxx = max(maxx, xv);
          miny = min(miny, yv); maxy = max(maxy, yv);
          const uint32_t tw = Tz[zv & 127];
          maxL = max(maxL, zv + 1 - (int)(tw >> 16));
          minW = min(minW, (int)(tw >> 16));
          xy[k] = ((uint32_t)xv & 0xFFFFu) | ((uint32_t)yv << 16);
          zc[k] = (uint32_t)zv & 0x7Fu;
          keyIn[e] = sort_key(sv);
          const float sf = __double2float_rn(sv);
          bb[k] = __float_as_uint(sf);
          if (!isinf(sf)) { const uint32_t fk = f32_key(sf); fmin = min(fmin, fk); fmax = max(fmax, fk); }
        }
      }
      const uint32_t word = __ballot_sync(0xFFFFFFFFu, keep);
      if (lane == 0) kbits[(k * THREADS >> 5) + warp] = word;
    }
    mode = __reduce_max_sync(0xFFFFFFFFu, mode);
    minz = __reduce_min_sync(0xFFFFFFFFu, minz);
    maxz = __reduce_max_sync(0xFFFFFFFFu, maxz);
    n_act = __reduce_add_sync(0xFFFFFFFFu, n_act);
    minx = __reduce_min_sync(0xFFFFFFFFu, minx); maxx = __reduce_max_sync(0xFFFFFFFFu, maxx);
    miny = __reduce_min_sync(0xFFFFFFFFu, miny); maxy = __reduce_max_sync(0xFFFFFFFFu, maxy);
    maxL = __reduce_max_sync(0xFFFFFFFFu, maxL); minW = __reduce_min_sync(0xFFFFFFFFu, minW);
    fmin = __reduce_min_sync(0xFFFFFFFFu, fmin); fmax = __reduce_max_sync(0xFFFFFFFFu, fmax);
    if (lane == 0) {
      atomicMax(&st->mode, mode); atomicMin(&st->minz, minz); atomicMax(&st->maxz, maxz);
      atomicAdd(&st->n_act, n_act);
      atomicMin(&st->minx, minx); atomicMax(&st->maxx, maxx);
      atomicMin(&st->miny, miny); atomicMax(&st->maxy, maxy);
      atomicMax(&st->maxL, maxL); atomicMin(&st->minW, minW);
      atomicMin(&st->fmin, fmin); atomicMax(&st->fmax, fmax);
      __threadfence_block();
      if (atomicAdd(&st->done, 1) == NW - 1) {
        // the last warp derives the frame's parameters once: eligibility (T_j >= 1 for every
        // active column <=> theta > 0 and no zero side), the reach L / R, the cell grid and
        // the score buckets
        volatile B2Stats* vs = st;
        const int na = vs->n_act;
        const int elig = vs->mode == kNarrow7 && (na == 0 || (a.theta > 0.0 && vs->minz >= 1));
        st->eligible = elig;
        const int L = vs->maxL, R = na > 0 ? vs->minW : 1;
        // cells Sx wide and Sy tall (any sides are exact).  Default: Sy = the power of two
        // nearest L + 1, Sx = Sy / 4, widened until the grid fits kMaxCells.
        int Sx, Sy;
        if (a.cell_q8 == 0) {
          const int h = L + 1;
          const int p2 = 1 << (31 - __clz(h));
          Sy = (long long)h * h > 2LL * p2 * p2 ? 2 * p2 : p2;
          Sx = Sy >> 2;
        } else {
          Sy = a.cell_q8 < 0 ? -a.cell_q8 : ((L + 1) * a.cell_q8 + 255) >> 8;
          Sx = Sy;
        }
        if (a.cell_sx > 0) Sx = a.cell_sx;
        Sx = max(Sx, kMinCellSide);
        Sy = max(Sy, kMinCellSide);
        int GX = 1, GY = 1;
        const int ox = vs->minx, oy = vs->miny;
        if (na > 0 && elig) {
          const int spx = vs->maxx - ox, spy = vs->maxy - oy;
          const bool p2 = (Sx & (Sx - 1)) == 0 && (Sy & (Sy - 1)) == 0;  // (widening keeps it)
          for (;;) {
            GX = (p2 ? spx >> (31 - __clz(Sx)) : spx / Sx) + 1;
            GY = (p2 ? spy >> (31 - __clz(Sy)) : spy / Sy) + 1;
            if ((long long)GX * GY <= Ly::kMaxCells) break;
            if (Sx < Sy) Sx *= 2;
            else { Sx *= 2; Sy *= 2; }
          }
        }
        st->L = L; st->R = R; st->GX = GX; st->GY = GY; st->cells = GX * GY; st->ox = ox; st->oy = oy;
        st->Mx = div_magic(Sx); st->My = div_magic(Sy);
        // value-linear score buckets over the finite fp32 range (monotone in the score, so
        // the in-bucket count on the full keys gives exact ranks)
        float smin = 0.0f, inv = 0.0f;
        if (vs->fmin <= vs->fmax) {
          smin = f32_unkey(vs->fmin);
          const float rng = __fsub_rn(f32_unkey(vs->fmax), smin);
          if (rng > 0.0f) inv = __fdiv_rn((float)NB, rng);
          if (isinf(inv)) inv = 0.0f;
        }
        st->smin = smin; st->inv = inv;
      }
    }
  }
  __syncthreads();
  PNMS_FRAME_TRACE(1);
  if (!st->eligible) {
    if (threadIdx.x == 0) binned_decline(a, f);
    return true;
  }
  const int n_act = st->n_act;
  const int L = st->L, R = st->R, GX = st->GX, GY = st->GY, cells = st->cells, ox = st->ox, oy = st->oy;
  const uint32_t Mx = st->Mx, My = st->My;
  {
    // ---- pass 2: cell and bucket histograms; the counters' old values are the arrival
    // ranks.  Bucket NB-1-floor((fl32(s) - smin) * inv): descending score = ascending key.
    const float smin = st->smin, inv = st->inv;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      if (zc[k] != 0xFFFFFFFFu) {
        const int ex = (int)(xy[k] & 0xFFFFu), ey = (int)(xy[k] >> 16);
        const int c = qdiv(ey - oy, My) * GX + qdiv(ex - ox, Mx);
        const uint32_t rc = atomic_inc_u16(comb, c);
        const float t = __fmul_rn(__fsub_rn(__uint_as_float(bb[k]), smin), inv);
        const int bi = t >= (float)NB ? NB - 1 : (t > 0.0f ? (int)t : 0);  // NaN (inv = 0, inf s): 0
        const int b = NB - 1 - bi;
        const uint32_t rb = atomic_inc_u16(comb, cells + b);
        zc[k] |= (rc << 7) | ((uint32_t)c << 19);  // z: 7 bits, cell rank: 12, cell: 13
        bb[k] = (uint32_t)b | (rb << 16);
      }
    }
  }
  __syncthreads();
  PNMS_FRAME_TRACE(2);
  // ---- exclusive scan over [cell counts | bucket counts | 0] (8 U4 counters per thread): cell
  // starts end in the sentinel n_act, bucket starts are offset by n_act; largest bucket
  {
    const int len = cells + NB + 1;
    constexpr int U4 = (Ly::kComb / 8 + THREADS - 1) / THREADS;  // uint4 (8 counters) per thread
    uint4* c4 = reinterpret_cast<uint4*>(comb) + threadIdx.x * U4;
    const int c0 = threadIdx.x * U4 * 8;
    uint32_t sum = 0, big = 0;
#pragma unroll
    for (int h = 0; h < U4; ++h) {
      if (c0 + 8 * h < len) {
        const uint4 v = c4[h];
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const uint32_t lo = w[t] & 0xFFFFu, hi = w[t] >> 16;
          sum += lo + hi;
          const int ci = c0 + 8 * h + 2 * t;
          if (ci >= cells) big = max(big, lo);
          if (ci + 1 >= cells) big = max(big, hi);
        }
      }
    }
    big = __reduce_max_sync(0xFFFFFFFFu, big);
    if (lane == 0) atomicMax(&st->big, (int)big);
    uint32_t run = block_exclusive_scan(sum, scan_tmp, nullptr);
#pragma unroll
    for (int h = 0; h < U4; ++h) {
      if (c0 + 8 * h < len) {
        const uint4 v = c4[h];
        uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const uint32_t lo = w[t] & 0xFFFFu, hi = w[t] >> 16;
          w[t] = run | ((run + lo) << 16);
          run += lo + hi;
        }
        c4[h] = make_uint4(w[0], w[1], w[2], w[3]);
      }
    }
  }
  __syncthreads();
  PNMS_FRAME_TRACE(3);
  if (st->big > kB2BucketMax) {
    if (threadIdx.x == 0) binned_decline(a, f);
    return true;
  }
  // ---- pass 3: keys and slots into bucket order
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    if (zc[k] != 0xFFFFFFFFu) {
      const int b = (int)(bb[k] & 0xFFFFu);
      const int pos = (int)comb[cells + b] - n_act + (int)(bb[k] >> 16);
      keyB[pos] = keyIn[threadIdx.x + k * THREADS];
      idxB[pos] = (uint16_t)(threadIdx.x + k * THREADS);
    }
  }
  __syncthreads();
  PNMS_FRAME_TRACE(4);
  // ---- pass 4: exact rank (count of the bucket's smaller keys), the record at the box's cell
  // position, and the box's candidate count (the records of the cells its window covers)
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    if (zc[k] != 0xFFFFFFFFu) {
      const int e = threadIdx.x + k * THREADS;
      const int b = (int)(bb[k] & 0xFFFFu);
      const int bs = (int)comb[cells + b] - n_act, be = (int)comb[cells + b + 1] - n_act;
      const uint64_t key = keyB[bs + (int)(bb[k] >> 16)];
      int rank = bs;
      for (int j = bs; j < be; ++j) {
        const uint64_t kj = keyB[j];
        rank += kj < key || (BY_INDEX && kj == key && (int)idxB[j] < e);
      }
      const int c = (int)(zc[k] >> 19);
      const int pos = (int)comb[c] + (int)((zc[k] >> 7) & 0xFFFu);
      const int32_t xv = (int32_t)(xy[k] & 0xFFFFu), yv = (int32_t)(xy[k] >> 16), zv = (int32_t)(zc[k] & 0x7Fu);
      const uint32_t T = Tz[zv] & 0xFFFFu;
      RecBin rb;
      rb.a = ((uint32_t)(xv + zv + 1) & 0xFFFFu) | ((uint32_t)(yv + zv + 1) << 16);
      rb.nb = ((uint32_t)(-xv) & 0xFFFFu) | ((uint32_t)(-yv) << 16);
      rb.w = -(int32_t)(T << 17) | (zv + 1);
      rb.k = (uint32_t)rank;
      recS[pos] = rb;
      idxS[pos] = (uint16_t)e;
      const int cx0 = qdiv(max(xv - L - ox, 0), Mx), cy0 = qdiv(max(yv - L - oy, 0), My);
      const int cx1 = min(GX - 1, qdiv(xv + zv + 1 - R - ox, Mx)), cy1 = min(GY - 1, qdiv(yv + zv + 1 - R - oy, My));
      int ncand = 0;
#pragma unroll
      for (int s = 0; s < kB2RunGroup; ++s) {
        const int yy = cy0 + s;
        if (yy <= cy1) ncand += (int)comb[yy * GX + cx1 + 1] - (int)comb[yy * GX + cx0];
      }
      for (int yy = cy0 + kB2RunGroup; yy <= cy1; ++yy) ncand += (int)comb[yy * GX + cx1 + 1] - (int)comb[yy * GX + cx0];
      const int cls = min(ncand, kB2RowClasses - 1);
      const uint32_t slot = atomicAdd(&rowhist[cls], 1u);
      xy[k] = (uint32_t)pos | ((uint32_t)cls << 12) | (slot << 18);
    }
  }
  __syncthreads();
  PNMS_FRAME_TRACE(5);
  // ---- rows into ascending candidate-count order (every warp scans the 64-class histogram)
  {
    const uint32_t h0 = rowhist[2 * lane], h1 = rowhist[2 * lane + 1];
    uint32_t inc = h0 + h1;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, inc, o);
      if (lane >= o) inc += t;
    }
    const uint32_t ex0 = inc - h0 - h1;  // start of class 2*lane; class 2*lane+1 starts at ex0 + h0
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const bool act = zc[k] != 0xFFFFFFFFu;
      const int cls = (int)((xy[k] >> 12) & 63u);
      const uint32_t s0 = __shfl_sync(0xFFFFFFFFu, ex0, cls >> 1);
      const uint32_t h0c = __shfl_sync(0xFFFFFFFFu, h0, cls >> 1);
      if (act) order[s0 + ((cls & 1) ? h0c : 0u) + (xy[k] >> 18)] = (uint16_t)(xy[k] & 0xFFFu);
    }
  }
  __syncthreads();
  PNMS_FRAME_TRACE(6);
  PNMS_FRAME_TRACE(7);
  // ---- scan: every row against every record of its window's cells (one run per cell row),
  // gate rank_j < rank_i; the runs of a row are walked as one flattened loop in groups of
  // kB2RunGroup cell rows
  unsigned long long tested = 0;
  const uint32_t rbase = static_cast<uint32_t>(__cvta_generic_to_shared(recS));
  for (int o = threadIdx.x; o < n_act; o += THREADS) {
    const int p = order[o];
    const uint4 ri = lds128(rbase + (uint32_t)p * 16u);  // a, nb, w, k
    const uint32_t zzi = __byte_perm(ri.z, 0u, 0x4040);   // (z+1, z+1)
    const int32_t ix = -(int32_t)(int16_t)(ri.y & 0xFFFFu), iy = -(int32_t)(int16_t)(ri.y >> 16);
    const int32_t iz = (int32_t)(ri.z & 0xFFu) - 1;
    const int cx0 = qdiv(max(ix - L - ox, 0), Mx), cy0 = qdiv(max(iy - L - oy, 0), My);
    const int cx1 = min(GX - 1, qdiv(ix + iz + 1 - R - ox, Mx)), cy1 = min(GY - 1, qdiv(iy + iz + 1 - R - oy, My));
    bool hit = false;
    for (int y0 = cy0; y0 <= cy1 && !hit; y0 += kB2RunGroup) {
      // runs s = 0..3 of cell rows y0 + s: item k of the group is record k + d_s for
      // c_s <= k < c_{s+1}
      int d[kB2RunGroup], c[kB2RunGroup + 1];
      c[0] = 0;
#pragma unroll
      for (int s = 0; s < kB2RunGroup; ++s) {
        const int yy = y0 + s;
        int qb = 0, qe = 0;
        if (yy <= cy1) { qb = comb[yy * GX + cx0]; qe = comb[yy * GX + cx1 + 1]; }
        d[s] = qb - c[s];
        c[s + 1] = c[s] + (qe - qb);
      }
      const int total = c[kB2RunGroup];
      int k = 0;
      bool go = total > 0;
      while (go) {
        int q = k + d[0];
        q = k >= c[1] ? k + d[1] : q;
        q = k >= c[2] ? k + d[2] : q;
        q = k >= c[3] ? k + d[3] : q;
        const uint4 g = lds128(rbase + (uint32_t)q * 16u);  // a, nb, w, k
        const uint32_t t1 = __viaddmin_s16x2(ri.x, g.y, zzi);
        const uint32_t t2 = __viaddmin_s16x2_relu(g.x, ri.y, t1);
        const uint32_t v = __vimin_s16x2_relu(t2, __byte_perm(g.z, 0u, 0x4040));
        if (COUNT) ++tested;
        hit = g.w < ri.w && (int)(v * v) + (int)g.z >= 0;
        ++k;
        go = !hit && k < total;
      }
    }
    if (hit) {
      const int i = idxS[p];
      atomicAnd(&kbits[i >> 5], ~(1u << (i & 31)));
    }
  }
  if (COUNT && a.pairs_tested) {
    tested = __reduce_add_sync(0xFFFFFFFFu, (unsigned)tested);
    if (lane == 0 && tested) atomicAdd(a.pairs_tested, tested);
  }
  __syncthreads();
  PNMS_FRAME_TRACE(8);
  // ---- compaction (engine.py:284-293): warp 0 scans the survivor words' popcounts, then every
  // thread writes the ascending keep indices of its own slots (coalesced)
  uint32_t* wpre = rowhist;  // [NP/32] word offsets (rowhist + scan_tmp: 128 entries)
  if (warp == 0) {
    constexpr int WPL = (NP / 32 + 31) / 32;  // words per lane
    const int W32 = a.W32;
    uint32_t c[WPL], sum = 0;
#pragma unroll
    for (int t = 0; t < WPL; ++t) {
      const int w = lane * WPL + t;
      const uint32_t bits = w < W32 && w < NP / 32 ? kbits[w] : 0u;
      if (a.keep_mask && w < W32) a.keep_mask[(long long)f * W32 + w] = bits;
      c[t] = __popc(bits);
      sum += c[t];
    }
    uint32_t inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, inc, o);
      if (lane >= o) inc += t;
    }
    uint32_t run = inc - sum;
#pragma unroll
    for (int t = 0; t < WPL; ++t) {
      if (lane * WPL + t < NP / 32) wpre[lane * WPL + t] = run;
      run += c[t];
    }
    if (lane == 31) {
      if (a.keep_count) a.keep_count[f] = (int32_t)inc;
      a.fallback[f] = 0;
    }
  }
  __syncthreads();
  if (a.keep_idx) {
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int e = threadIdx.x + k * THREADS;
      const uint32_t bits = kbits[e >> 5];
      if ((bits >> lane) & 1u) a.keep_idx[fbase + wpre[e >> 5] + __popc(bits & lanemask_lt())] = e;
    }
  }
  PNMS_FRAME_TRACE(9);
  return false;
}

template <bool BY_INDEX, bool COUNT, int PER, int THREADS, int MINB = (THREADS == 512 ? 3 : 1)>
__global__ void __launch_bounds__(THREADS, MINB) pnms_binned2_frame(BinArgs a) {
  binned2_frame_body<BY_INDEX, COUNT, PER, THREADS>(a);
}

}  // namespace pnms

// pnms_binned_pairs.cuh — exact spatially binned NMS as a cell-pair tile sweep, one CTA per
// frame, everything in shared memory.  Same eligibility, cells and result as
// pnms_binned_frame (pnms_binned.cuh); a different enumeration of the work.
//
// Every unordered pair of boxes that can overlap lies in one cell or in two neighbouring
// cells.  Cell c visits the pairs (row in c) x (column in c's half neighbourhood): its own
// cell (columns after the row only), E, and the cell row below SW, S, SE.  In row-major cell
// order {self, E} and {SW, S, SE} are two contiguous position ranges, so the pairs of one
// cell form a dense rows x columns tile that a warp sweeps with one pair per lane (no
// per-cell sort, no data-dependent loop per row).  Per pair the reference's gate
// (engine.py:233-235) decides which box, if any, can suppress the other — at most one
// direction passes — and the suppression test (engine.py:219-232, w*h >= T_j of the
// outranking box j) marks the outranked box.  Every overlapping pair is visited exactly once,
// so a box is suppressed iff the reference's row AND clears it.
#pragma once
#include "pnms_binned.cuh"

namespace pnms {

constexpr int kPairThreads = 512;
constexpr int kPairWarps = kPairThreads / 32;

// Pair record (16 B): narrow7 geometry and threshold of RecBin, plus the input slot.
//   a = (x+z+1, y+z+1), nb = (-x, -y), w = -(T << 17) | (z+1), idx = input slot
struct __align__(16) RecPair {
  uint32_t a, nb;
  int32_t w;
  uint32_t idx;
};

inline size_t binned_pairs_smem_bytes(int npad) {
  return (size_t)npad * (sizeof(RecPair) + 8) + (size_t)(binned_max_cells(npad) + 4) * 4 + (size_t)(npad / 32 + 4) * 4 * 2 +
         64 * 4 + sizeof(BinStats) + 64;
}

template <bool BY_INDEX, bool COUNT, int PER>
__global__ void __launch_bounds__(kPairThreads, (PER == 4 ? 3 : 1)) pnms_binned_pairs_frame(BinArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int f = blockIdx.x;
  const long long fbase = (long long)f * a.n_max;
  const int cnt = frame_count(a.counts, f, a.n_max);
  const int npad = binned_npad(a.n_max);
  // the fallback kernels over the declined-frame list may launch once every CTA has started
  // (programmatic dependent launch); they wait for this grid's completion before reading
  pdl_trigger();
  RecPair* recS = reinterpret_cast<RecPair*>(smem_raw);                    // [npad] cell order
  uint64_t* keyS = reinterpret_cast<uint64_t*>(recS + npad);               // [npad] sort keys
  const int max_cells = binned_max_cells(npad);
  uint32_t* cstart = reinterpret_cast<uint32_t*>(keyS + npad);             // [cells+2]
  uint32_t* kbits = cstart + max_cells + 4;                                // [npad/32] survivors, input order
  uint32_t* sbits = kbits + npad / 32 + 4;                                 // [npad/32] suppressed, cell order
  uint32_t* scan_tmp = sbits + npad / 32 + 4;                              // [64]
  BinStats* st = reinterpret_cast<BinStats*>(scan_tmp + 64);

  if (threadIdx.x == 0) {
    st->mode = kNarrow7; st->minz = 0x7FFFFFFF; st->maxz = 0;
    st->minx = st->miny = 0x7FFFFFFF; st->maxx = st->maxy = -0x7FFFFFFF;
    st->big = 0; st->n_act = 0;
  }
  for (int w = threadIdx.x; w < npad / 32; w += kPairThreads) { kbits[w] = 0u; sbits[w] = 0u; }
  __syncthreads();
  if (a.n_max > PER * kPairThreads) {
    if (threadIdx.x == 0) binned_decline(a, f);
    return;
  }
  // ---- pass 1: the frame from HBM once, kept in registers; frame statistics
  uint32_t xy[PER], zc[PER];
  {
    int mode = kNarrow7, minz = 0x7FFFFFFF, maxz = 0, n_act = 0;
    int minx = 0x7FFFFFFF, miny = 0x7FFFFFFF, maxx = -0x7FFFFFFF, maxy = -0x7FFFFFFF;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int e = threadIdx.x + k * kPairThreads;
      xy[k] = 0u; zc[k] = 0xFFFFFFFFu;
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
          atomicOr(&kbits[e >> 5], 1u << (e & 31));  // NaN: never gated, never suppresses
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
  const int n_act = st->n_act;
  const bool eligible = st->mode == kNarrow7 && (n_act == 0 || (a.theta > 0.0 && st->minz >= 1));
  if (!eligible) {
    if (threadIdx.x == 0) binned_decline(a, f);
    return;
  }
  int S = st->maxz + 1, GX = 1, GY = 1;
  const int ox = st->minx, oy = st->miny;
  if (n_act > 0) {
    for (;;) {
      GX = (st->maxx - ox) / S + 1;
      GY = (st->maxy - oy) / S + 1;
      if ((long long)GX * GY <= max_cells) break;
      S *= 2;
    }
  }
  const uint32_t M = div_magic(S);
  const int cells = GX * GY;
  for (int c = threadIdx.x; c < cells + 2; c += kPairThreads) cstart[c] = 0u;
  __syncthreads();
  // ---- pass 2: histogram (the atomic's return value is the box's slot inside its cell)
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    if (zc[k] != 0xFFFFFFFFu) {
      const int ex = (int)(xy[k] & 0xFFFFu), ey = (int)(xy[k] >> 16);
      const int c = qdiv(ey - oy, M) * GX + qdiv(ex - ox, M);
      const uint32_t r = atomicAdd(&cstart[c], 1u);
      zc[k] |= ((uint32_t)c << 16) | (min(r, 255u) << 8);
    }
  }
  __syncthreads();
  {
    const int per = (cells + kPairThreads - 1) / kPairThreads;
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
    if (threadIdx.x == 0) { cstart[cells] = n_act; cstart[cells + 1] = n_act; }
  }
  __syncthreads();
  if (st->big > kBinCellMax) {
    if (threadIdx.x == 0) binned_decline(a, f);
    return;
  }
  // ---- pass 3: records and keys straight into cell order (unsorted inside a cell)
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    if (zc[k] != 0xFFFFFFFFu) {
      const int e = threadIdx.x + k * kPairThreads;
      const uint32_t pos = cstart[zc[k] >> 16] + ((zc[k] >> 8) & 0xFFu);
      const int32_t xv = (int32_t)(xy[k] & 0xFFFFu), yv = (int32_t)(xy[k] >> 16), zv = (int32_t)(zc[k] & 0xFFu);
      const RecNarrow rn = make_rec_narrow(xv, yv, zv, a.theta, kNarrow7);
      RecPair rp;
      rp.a = rn.a; rp.nb = rn.nb; rp.w = rn.negT | (zv + 1); rp.idx = (uint32_t)e;
      recS[pos] = rp;
      keyS[pos] = sort_key(a.s[fbase + e]);
    }
  }
  __syncthreads();
  // ---- pair tiles: warp w sweeps cells w, w + 16, ...; lane = one (row, column) pair
  unsigned long long tested = 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float fGX = (float)GX;
  for (int c = warp; c < cells; c += kPairWarps) {
    const int r0 = (int)cstart[c], m = (int)cstart[c + 1] - r0;
    if (m == 0) continue;
    const int cy = (int)(((float)c + 0.5f) / fGX), cx = c - cy * GX;
    const int a1 = (int)cstart[cx + 1 < GX ? c + 2 : c + 1];          // self + E
    int b0 = 0, b1 = 0;
    if (cy + 1 < GY) {                                                 // SW, S, SE
      b0 = (int)cstart[c + GX - (cx > 0 ? 1 : 0)];
      b1 = (int)cstart[c + GX + (cx + 1 < GX ? 2 : 1)];
    }
    const int nA = a1 - r0, ncols = nA + (b1 - b0), total = m * ncols;
    const float inv = 1.0f / (float)ncols;
    for (int k = lane; k < total; k += 32) {
      // exact: k < 2^16 and ncols <= 9 * 64, far from the float rounding limit
      const int row = (int)(((float)k + 0.5f) * inv);
      const int col = k - row * ncols;
      const int i = r0 + row;
      const int j = col < nA ? r0 + col : b0 + (col - nA);
      if (j <= i) continue;                                            // own cell: each pair once
      const RecPair ri = recS[i], rj = recS[j];
      const uint64_t ki = keyS[i], kj = keyS[j];
      // the reference's gate: which of the two may suppress the other (at most one)
      bool i_loses = kj < ki, j_loses = ki < kj;
      if (BY_INDEX && ki == kj) { i_loses = ri.idx > rj.idx; j_loses = !i_loses; }
      if (!(i_loses | j_loses)) continue;
      if (COUNT) ++tested;
      const uint32_t t1 = __viaddmin_s16x2(ri.a, rj.nb, __byte_perm((uint32_t)ri.w, 0u, 0x4040));
      const uint32_t t2 = __viaddmin_s16x2_relu(rj.a, ri.nb, t1);
      const uint32_t v = __vimin_s16x2_relu(t2, __byte_perm((uint32_t)rj.w, 0u, 0x4040));
      const int tw = i_loses ? rj.w : ri.w;                             // threshold of the winner
      if ((int)(v * v) + tw >= 0) {
        const int loser = i_loses ? i : j;
        atomicOr(&sbits[loser >> 5], 1u << (loser & 31));
      }
    }
  }
  if (COUNT && a.pairs_tested) {
    tested = __reduce_add_sync(0xFFFFFFFFu, (unsigned)tested);
    if (lane == 0 && tested) atomicAdd(a.pairs_tested, tested);
  }
  __syncthreads();
  // ---- survivors in input order (+ the implicit padding gate, engine.py:233: s < 0 drops)
  const bool pad_rule = a.d_max > cnt;
  for (int p = threadIdx.x; p < n_act; p += kPairThreads) {
    if ((sbits[p >> 5] >> (p & 31)) & 1u) continue;
    const int i = (int)recS[p].idx;
    if (pad_rule && a.s[fbase + i] < 0.0) continue;
    atomicOr(&kbits[i >> 5], 1u << (i & 31));
  }
  __syncthreads();
  // ---- compaction (engine.py:284-293)
  const int words_per_thread = (a.W32 + kPairThreads - 1) / kPairThreads;
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

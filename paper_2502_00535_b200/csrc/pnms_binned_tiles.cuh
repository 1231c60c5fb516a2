// pnms_binned_tiles.cuh — single-frame latency path for large frames (4096 < n, small batches):
// the exact binned NMS of pnms_binned.cuh spread over kTilesPerFrame independent CTAs per
// frame, with no inter-CTA communication until the survivor mask.
//
// Every CTA of a frame streams the whole frame from L2 (it is tiny next to a CTA's work:
// 20 B per slot), computes the same frame statistics, cells of side max_z + 1 and tile
// layout, and then owns one rectangular tile of cells.  It bins the boxes of its tile and of
// the one-cell halo around it (a row's reach adds at most one cell on every side), orders its
// cells, scans the rows of its tile exactly like pnms_binned_frame (gate-prefix skip, exact
// rescan on equal key halves) and sets the survivors' bits in the frame's global mask.
// pnms_mask_compact then turns the mask into ascending keep indices.  A frame is declined
// (dense pipeline) if it is ineligible or a tile region exceeds kTileCap boxes / a cell
// exceeds kBinCellMax boxes.
#pragma once
#include "pnms_binned.cuh"

namespace pnms {

constexpr int kTileThreads = 512;
constexpr int kTilesPerFrame = 128;
constexpr int kTileCap = 3072;       // boxes of tile + halo a CTA may hold
constexpr int kTileCells = 1024;     // cells of tile + halo a CTA may hold

struct TileArgs {
  BinArgs b;
  uint32_t* mask;        // [batch][W32] survivor bits: zero at entry, zeroed again by pnms_mask_compact
  int* decline;          // [batch] set by any CTA of a frame that must go to the dense path (ditto)
};

inline size_t binned_tiles_smem_bytes() {
  return (size_t)kTileCap * (sizeof(RecBin) + 8 + 2 + 2 + 4 + 8 + 2 + 6) + (size_t)(kTileCells + 4) * 4 + 64 * 4 +
         sizeof(BinStats) + 64;
}

template <bool BY_INDEX>
__global__ void __launch_bounds__(kTileThreads, 1) pnms_binned_tiles(TileArgs ta) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const BinArgs& a = ta.b;
  const int f = blockIdx.x / kTilesPerFrame, t = blockIdx.x % kTilesPerFrame;
  const long long fbase = (long long)f * a.n_max;
  const int cnt = frame_count(a.counts, f, a.n_max);
  pdl_trigger();  // pnms_mask_compact may launch early (PDL)
  unsigned long long* trace = a.trace;          // diagnostics: per-CTA phase timestamps
#define PNMS_TILE_TRACE(ph)                                                               \
  do {                                                                                    \
    if (trace && threadIdx.x == 0 && t < 16) {                                            \
      unsigned long long t_;                                                              \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                              \
      trace[t * 16 + (ph)] = t_;                                                          \
    }                                                                                     \
  } while (0)
  PNMS_TILE_TRACE(0);
  RecBin* recS = reinterpret_cast<RecBin*>(smem_raw);
  uint64_t* keyS = reinterpret_cast<uint64_t*>(recS + kTileCap);
  uint16_t* idxS = reinterpret_cast<uint16_t*>(keyS + kTileCap);
  uint16_t* cellS = idxS + kTileCap;                                        // local cell of position p
  uint32_t* lst = reinterpret_cast<uint32_t*>(cellS + kTileCap);           // region boxes: slot | cell<<16 ...
  uint64_t* tKey = reinterpret_cast<uint64_t*>(lst + kTileCap);            // arrival-order keys ...
  uint16_t* tIdx = reinterpret_cast<uint16_t*>(tKey + kTileCap);           // ... and slots (cell-grouped)
  uint32_t* cstart = reinterpret_cast<uint32_t*>(tIdx + 4 * kTileCap);
  uint32_t* scan_tmp = cstart + kTileCells + 4;
  BinStats* st = reinterpret_cast<BinStats*>(scan_tmp + 64);
  __shared__ int s_n;
  __shared__ uint32_t s_big;

  if (threadIdx.x == 0) {
    st->mode = kNarrow7; st->minz = 0x7FFFFFFF; st->maxz = 0;
    st->minx = st->miny = 0x7FFFFFFF; st->maxx = st->maxy = -0x7FFFFFFF;
    st->big = 0; st->n_act = 0; st->maxL = 0; st->minW = 0x7FFFFFFF;
    s_n = 0; s_big = 0;
  }
  // T_z | wmin_z << 16 (pnms_binned2.cuh): the theta reach of a suppressing column
  __shared__ uint32_t Tz[128];
  if (threadIdx.x < 128) {
    const int zv = threadIdx.x;
    const uint32_t T = zv == 0 ? 0u : (uint32_t)ceil(ref_threshold(a.theta, zv));
    Tz[zv] = T | (((T + zv) / (uint32_t)(zv + 1)) << 16);
  }
  for (int c = threadIdx.x; c < kTileCells + 4; c += kTileThreads) cstart[c] = 0u;
  __syncthreads();
  // ---- pass 1: frame statistics over every slot (identical in every CTA of the frame).  The
  // frame is streamed from L2 by every CTA: 16 B vector loads, several in flight per thread.
  const bool vec = ((fbase & 3) == 0) && ((((uintptr_t)a.x) | ((uintptr_t)a.y) | ((uintptr_t)a.z) | ((uintptr_t)a.s)) & 15) == 0;
  {
    int mode = kNarrow7, minz = 0x7FFFFFFF, maxz = 0, n_act = 0, maxL = 0, minW = 0x7FFFFFFF;
    int minx = 0x7FFFFFFF, miny = 0x7FFFFFFF, maxx = -0x7FFFFFFF, maxy = -0x7FFFFFFF;
    auto visit = [&](int e, int32_t xv, int32_t yv, int32_t zv, double sv) {
      mode = max(mode, frame_mode_of(xv, yv, zv));
      if (sv == sv) {
        ++n_act;
        minz = min(minz, zv); maxz = max(maxz, zv);
        minx = min(minx, xv); maxx = max(maxx, xv);
        miny = min(miny, yv); maxy = max(maxy, yv);
        const uint32_t tw = Tz[zv & 127];
        maxL = max(maxL, zv + 1 - (int)(tw >> 16)); minW = min(minW, (int)(tw >> 16));
      } else if (t == 0) {
        atomicOr(ta.mask + (long long)f * a.W32 + (e >> 5), 1u << (e & 31));  // NaN: survivor
      }
    };
    const int nv = vec ? cnt / 4 : 0;
    // every CTA of the frame streams the same lines: start each at a different offset so the
    // requests spread over the L2 slices instead of hammering the same lines together
    const int rot = (int)(((long long)t * nv) / kTilesPerFrame);
#pragma unroll 4
    for (int vv = threadIdx.x; vv < nv; vv += kTileThreads) {
      const int v = vv + rot < nv ? vv + rot : vv + rot - nv;
      const long long g = fbase + 4LL * v;
      const int4 X = *reinterpret_cast<const int4*>(a.x + g), Y = *reinterpret_cast<const int4*>(a.y + g);
      const int4 Z = *reinterpret_cast<const int4*>(a.z + g);
      const double2 S0 = *reinterpret_cast<const double2*>(a.s + g), S1 = *reinterpret_cast<const double2*>(a.s + g + 2);
      visit(4 * v, X.x, Y.x, Z.x, S0.x);
      visit(4 * v + 1, X.y, Y.y, Z.y, S0.y);
      visit(4 * v + 2, X.z, Y.z, Z.z, S1.x);
      visit(4 * v + 3, X.w, Y.w, Z.w, S1.y);
    }
    for (int e = 4 * nv + threadIdx.x; e < cnt; e += kTileThreads) {
      const long long g = fbase + e;
      visit(e, a.x[g], a.y[g], a.z[g], a.s[g]);
    }
    mode = __reduce_max_sync(0xFFFFFFFFu, mode);
    minz = __reduce_min_sync(0xFFFFFFFFu, minz);
    maxz = __reduce_max_sync(0xFFFFFFFFu, maxz);
    maxL = __reduce_max_sync(0xFFFFFFFFu, maxL); minW = __reduce_min_sync(0xFFFFFFFFu, minW);
    n_act = __reduce_add_sync(0xFFFFFFFFu, n_act);
    minx = __reduce_min_sync(0xFFFFFFFFu, minx); maxx = __reduce_max_sync(0xFFFFFFFFu, maxx);
    miny = __reduce_min_sync(0xFFFFFFFFu, miny); maxy = __reduce_max_sync(0xFFFFFFFFu, maxy);
    if ((threadIdx.x & 31) == 0) {
      atomicMax(&st->mode, mode); atomicMin(&st->minz, minz); atomicMax(&st->maxz, maxz);
      atomicMax(&st->maxL, maxL); atomicMin(&st->minW, minW);
      atomicAdd(&st->n_act, n_act);
      atomicMin(&st->minx, minx); atomicMax(&st->maxx, maxx);
      atomicMin(&st->miny, miny); atomicMax(&st->maxy, maxy);
    }
  }
  __syncthreads();
  PNMS_TILE_TRACE(1);
  const int n_act = st->n_act;
  const bool eligible = st->mode == kNarrow7 && (n_act == 0 || (a.theta > 0.0 && st->minz >= 1));
  if (!eligible) {
    if (t == 0 && threadIdx.x == 0) ta.decline[f] = 1;
    return;
  }
  if (n_act == 0) return;
  // ---- cells Sy = max_z + 1 tall and Sx = Sy / 4 wide (as pnms_binned.cuh: fewer runs per
  // row, tight x ranges) and a tile layout of at most kTilesPerFrame tiles, square in pixels
  // the theta reach (pnms_binned2.cuh): a suppressing column's corner lies within
  // [x - L, x + z + 1 - R] (same for y); cells taller than either vertical reach (a one-row halo)
  const int g_L = st->maxL, g_R = st->minW;
  const int Sy = max(max(g_L, st->maxz + 1 - g_R) + 1, kMinCellSide), Sx = max(Sy >> 2, kMinCellSide);
  const int ox = st->minx, oy = st->miny;
  const uint32_t Mx = div_magic(Sx), My = div_magic(Sy);
  const int GX = (st->maxx - ox) / Sx + 1, GY = (st->maxy - oy) / Sy + 1;
  // halo columns: a row reaches L pixels left and z + 1 - R right
  const int hxl = (g_L + Sx - 1) / Sx, hxr = (st->maxz + 1 - g_R + Sx - 1) / Sx;
  int TX = (int)sqrtf((float)kTilesPerFrame * (float)(GX * Sx) / (float)(GY * Sy) + 0.5f);
  TX = max(1, min(TX, min(GX, kTilesPerFrame)));
  int TY = max(1, min(GY, kTilesPerFrame / TX));
  const int tw = (GX + TX - 1) / TX, th = (GY + TY - 1) / TY;
  TX = (GX + tw - 1) / tw;
  TY = (GY + th - 1) / th;
  if (t >= TX * TY) return;
  const int tx = t % TX, ty = t / TX;
  const int cx0 = max(tx * tw - hxl, 0), cx1 = min((tx + 1) * tw - 1 + hxr, GX - 1);  // region incl. halo
  const int cy0 = max(ty * th - 1, 0), cy1 = min((ty + 1) * th, GY - 1);
  const int ix0 = tx * tw, ix1 = min((tx + 1) * tw, GX) - 1;              // interior (own rows)
  const int iy0 = ty * th, iy1 = min((ty + 1) * th, GY) - 1;
  const int LW = cx1 - cx0 + 1, LH = cy1 - cy0 + 1, lcells = LW * LH;
  if (lcells + 1 > kTileCells) {
    if (threadIdx.x == 0) ta.decline[f] = 1;
    return;
  }
  // ---- pass 2: the region's boxes (L2-resident re-read of x, y; NaN rows have no cell)
  {
    const bool has_nan = n_act != cnt;
    // the region in pixels: most boxes are rejected by four compares, no cell arithmetic
    const int px0 = ox + cx0 * Sx, px1 = ox + (cx1 + 1) * Sx - 1;
    const int py0 = oy + cy0 * Sy, py1 = oy + (cy1 + 1) * Sy - 1;
    auto take = [&](int e, int32_t xv, int32_t yv) {
      bool in = xv >= px0 && xv <= px1 && yv >= py0 && yv <= py1;
      if (!in) return;                                     // ~98 % of the frame
      if (has_nan && a.s[fbase + e] != a.s[fbase + e]) return;  // NaN rows have no cell
      const int slot = atomicAdd(&s_n, 1);
      const int lc = (qdiv(yv - oy, My) - cy0) * LW + (qdiv(xv - ox, Mx) - cx0);
      const uint32_t r = atomicAdd(&cstart[lc], 1u);
      if (slot < kTileCap) {
        lst[slot] = (uint32_t)e | ((uint32_t)lc << 16);  // e < 65536, lc < kTileCells
        cellS[slot] = (uint16_t)min(r, 65535u);          // rank in the cell, consumed below
      }
    };
    const int nv = vec ? cnt / 4 : 0;
    const int rot = (int)(((long long)t * nv) / kTilesPerFrame);
#pragma unroll 4
    for (int vv = threadIdx.x; vv < nv; vv += kTileThreads) {
      const int v = vv + rot < nv ? vv + rot : vv + rot - nv;
      const long long g = fbase + 4LL * v;
      const int4 X = *reinterpret_cast<const int4*>(a.x + g), Y = *reinterpret_cast<const int4*>(a.y + g);
      take(4 * v, X.x, Y.x);
      take(4 * v + 1, X.y, Y.y);
      take(4 * v + 2, X.z, Y.z);
      take(4 * v + 3, X.w, Y.w);
    }
    for (int e = 4 * nv + threadIdx.x; e < cnt; e += kTileThreads) take(e, a.x[fbase + e], a.y[fbase + e]);
  }
  __syncthreads();
  PNMS_TILE_TRACE(2);
  const int nreg = s_n;
  {
    const int per = (lcells + kTileThreads - 1) / kTileThreads;
    const int b0 = threadIdx.x * per;
    uint32_t sum = 0, big = 0;
    for (int q = 0; q < per; ++q) {
      const int c = b0 + q;
      if (c < lcells) { sum += cstart[c]; big = max(big, cstart[c]); }
    }
    big = __reduce_max_sync(0xFFFFFFFFu, big);
    if ((threadIdx.x & 31) == 0) atomicMax(&s_big, big);
    uint32_t run = block_exclusive_scan(sum, scan_tmp, nullptr);
    for (int q = 0; q < per; ++q) {
      const int c = b0 + q;
      if (c < lcells) { const uint32_t v = cstart[c]; cstart[c] = run; run += v; }
    }
    if (threadIdx.x == 0) cstart[lcells] = (uint32_t)min(nreg, kTileCap);
  }
  __syncthreads();
  if (nreg > kTileCap || s_big > (uint32_t)kBinCellMax) {
    if (threadIdx.x == 0) ta.decline[f] = 1;
    return;
  }
  // ---- pass 3: keys into arrival order (cell-grouped), then every box counts the members of
  // its cell that precede it in (key, slot) order and lands at its final position — no serial
  // per-cell sort on the latency path
  uint16_t rank_of[kTileCap / kTileThreads];
#pragma unroll
  for (int k = 0; k < kTileCap / kTileThreads; ++k) {
    const int q = threadIdx.x + k * kTileThreads;
    rank_of[k] = q < nreg ? cellS[q] : 0;
  }
#pragma unroll
  for (int k = 0; k < kTileCap / kTileThreads; ++k) {
    const int q = threadIdx.x + k * kTileThreads;
    if (q >= nreg) continue;
    const int e = (int)(lst[q] & 0xFFFFu), lc = (int)(lst[q] >> 16);
    const uint32_t pa = cstart[lc] + rank_of[k];
    tKey[pa] = sort_key(a.s[fbase + e]);
    tIdx[pa] = (uint16_t)e;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kTileCap / kTileThreads; ++k) {
    const int q = threadIdx.x + k * kTileThreads;
    if (q >= nreg) continue;
    const int e = (int)(lst[q] & 0xFFFFu), lc = (int)(lst[q] >> 16);
    const int b = (int)cstart[lc], en = (int)cstart[lc + 1];
    const uint64_t key = tKey[b + rank_of[k]];
    int rank = 0;
    for (int j = b; j < en; ++j) {
      const uint64_t kj = tKey[j];
      rank += kj < key || (kj == key && (int)tIdx[j] < e);
    }
    const int pos = b + rank;
    const long long g = fbase + e;
    const int32_t xv = a.x[g], yv = a.y[g], zv = a.z[g];
    const RecNarrow rn = make_rec_narrow(xv, yv, zv, a.theta, kNarrow7);
    RecBin rb;
    rb.a = rn.a; rb.nb = rn.nb; rb.w = rn.negT | (zv + 1) | ((en - pos) << 8); rb.k = (uint32_t)(key >> 32);
    recS[pos] = rb;
    keyS[pos] = key;
    idxS[pos] = (uint16_t)e;
  }
  __syncthreads();
  // local cell of every position (for the interior test of the row scan)
  for (int c = threadIdx.x; c < lcells; c += kTileThreads)
    for (int i = (int)cstart[c]; i < (int)cstart[c + 1]; ++i) cellS[i] = (uint16_t)c;
  __syncthreads();
  PNMS_TILE_TRACE(4);
  // ---- rows of the interior cells against their reachable cells (all inside the region)
  const bool pad_rule = a.d_max > cnt;
  const int nl = (int)cstart[lcells];
  const uint32_t rbase = static_cast<uint32_t>(__cvta_generic_to_shared(recS));
  for (int p = threadIdx.x; p < nl; p += kTileThreads) {
    const int lc = cellS[p];
    const int gcx = cx0 + lc % LW, gcy = cy0 + lc / LW;
    if (gcx < ix0 || gcx > ix1 || gcy < iy0 || gcy > iy1) continue;  // halo box: another tile's row
    const RecBin ri = recS[p];
    const uint32_t zzi = __byte_perm((uint32_t)ri.w, 0u, 0x4040);
    const int32_t ix = -(int32_t)(int16_t)(ri.nb & 0xFFFFu), iy = -(int32_t)(int16_t)(ri.nb >> 16);
    const int32_t iz = (int32_t)(ri.w & 0xFF) - 1;
    const int rx0 = max(qdiv(max(ix - g_L - ox, 0), Mx), cx0), ry0 = max(qdiv(max(iy - g_L - oy, 0), My), cy0);
    const int rx1 = min(cx1, qdiv(ix + iz + 1 - g_R - ox, Mx)), ry1 = min(cy1, qdiv(iy + iz + 1 - g_R - oy, My));
    const uint32_t pb = rbase + (uint32_t)p * (uint32_t)sizeof(RecBin);
    bool sup = false;
    unsigned long long tested = 0;
    for (int yy = ry0; yy <= ry1 && !sup; ++yy) {
      const int lr = (yy - cy0) * LW - cx0;
      const uint32_t qb = rbase + cstart[lr + rx0] * (uint32_t)sizeof(RecBin);
      const uint32_t qe = rbase + cstart[lr + rx1 + 1] * (uint32_t)sizeof(RecBin);
      sup = binned_scan_run<BY_INDEX, false>(rbase, qb, qe, ri, zzi, pb, keyS, idxS, p, tested);
    }
    const int i = idxS[p];
    if (!sup && pad_rule && a.s[fbase + i] < 0.0) sup = true;
    if (!sup) atomicOr(ta.mask + (long long)f * a.W32 + (i >> 5), 1u << (i & 31));
  }
  __syncthreads();
  PNMS_TILE_TRACE(5);
#undef PNMS_TILE_TRACE
}

// survivor mask -> ascending keep indices, count and mask output (engine.py:284-293); one CTA
// per frame; frames flagged in `decline` are left to the dense pipeline.  The mask and flag
// live in the caller's persistent zeroed scratch: every word is zeroed again by the thread
// that read it last, so the next call needs no memset.
__global__ void __launch_bounds__(512) pnms_mask_compact(TileArgs ta) {
  pdl_wait();  // PDL: the tile kernel's mask is complete after this
  const BinArgs& a = ta.b;
  const int f = blockIdx.x;
  __shared__ uint32_t scan_tmp[64];
  uint32_t* m = ta.mask + (long long)f * a.W32;
  const int wpt = (a.W32 + 511) / 512;
  const int w0 = threadIdx.x * wpt, w1 = min(w0 + wpt, a.W32);
  const int declined = ta.decline[f];
  __syncthreads();  // every thread has the flag before thread 0 clears it
  if (declined) {
    for (int w = w0; w < w1; ++w) m[w] = 0u;
    if (threadIdx.x == 0) {
      ta.decline[f] = 0;
      binned_decline(a, f);
    }
    return;
  }
  const long long fbase = (long long)f * a.n_max;
  uint32_t local = 0;
  for (int w = w0; w < w1; ++w) {
    const uint32_t bits = m[w];
    local += __popc(bits);
    if (a.keep_mask) a.keep_mask[(long long)f * a.W32 + w] = bits;
  }
  uint32_t total;
  uint32_t pos = block_exclusive_scan(local, scan_tmp, &total);
  for (int w = w0; w < w1; ++w) {
    uint32_t bits = m[w];
    m[w] = 0u;
    if (a.keep_idx) {
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

// pnms_coop.cuh — latency path for single large frames: one cooperative launch of T CTAs per
// frame (all co-resident) that share the frame-level work through global memory instead of
// repeating it in every CTA (pnms_binned_tiles.cuh streams the whole frame into each of its
// 128 CTAs twice).
//
//   phase 0  CTA r reads its slice of the frame once: statistics into the frame's global
//            accumulators (shared-memory reduction, one atomic per field per CTA); NaN rows
//            are survivors (their mask bits are set here)
//   barrier
//   phase 1  every CTA derives the same parameters (eligibility, the theta reach L / R of
//            pnms_binned2.cuh, cells, a tile layout of T tiles with halos covering the reach)
//            and appends each box of its slice to the list of every tile whose region (tile
//            plus halo) holds the box's cell: one 16 B entry {x|y<<16, z|dead<<7|slot<<16, key}
//   barrier
//   phase 2  CTA r owns tile r: its region's entries into shared memory, a counting sort into
//            the region's cells, 16 B records plus the 64-bit keys at the cell positions, and
//            the rows of the tile's interior scanned against their windows with the
//            reference's gate on the full keys (engine.py:233-235; the input slot breaks
//            by_index ties); survivor bits into the frame's global mask
//   barrier
//   phase 3  CTA r compacts mask words [r*wpc, (r+1)*wpc) into ascending keep indices (its
//            offset = popcount of the words before it); the last CTA to finish re-zeroes the
//            frame's scratch for the next call
//
// Exactness is that of pnms_binned2.cuh: every column that can clear row i's bit lies in i's
// window, the window of an interior row lies inside the tile's region, and the gate compares
// the frame's own 64-bit keys.  A frame is declined (dense pipeline, through the device-side
// list) if it is not eligible or a tile region exceeds kCoopCap boxes.
#pragma once
#include "pnms_binned2.cuh"

namespace pnms {

constexpr int kCoopThreads = 256;
constexpr int kCoopCap = 1024;          // region entries a tile CTA holds
constexpr int kCoopCells = 2048;        // region cells a tile CTA holds
constexpr int kCoopMaxFrames = 2;       // frames per call (latency path)
constexpr int kCoopMaxTiles = 512;
constexpr int kCoopBoxesPerTile = 128;  // default tile count: one tile per this many slots

// per-frame scratch in the caller's persistent zeroed workspace head; every field's identity
// is 0 (minima are kept as maxima of complements), and the last CTA re-zeroes it all
struct CoopFrame {
  uint32_t mode, nminz, maxz, nminx, nminy, maxx, maxy, n_act;  // ox(v) = v ^ 2^31: signed order
  uint32_t maxL, nminW, pad0, pad1;
  uint32_t barrier, done, overflow, big;
  uint32_t tile_cnt[kCoopMaxTiles];
};
static_assert(sizeof(CoopFrame) % 16 == 0, "CoopFrame layout");
__host__ __device__ constexpr size_t coop_scratch_bytes(int n_max) {
  return (size_t)kCoopMaxFrames * (sizeof(CoopFrame) + (size_t)((n_max + 127) / 128) * 16);
}

struct CoopArgs {
  BinArgs b;
  CoopFrame* scr;      // [kCoopMaxFrames] frame scratch (zero at entry, zero at exit)
  uint32_t* mask;      // [kCoopMaxFrames][W32 rounded to 4] survivor bits (zero at entry and exit)
  uint4* lists;        // [batch][T][cap] tile entries
  int tiles;           // T: CTAs per frame
  int cap;             // entries per tile list
};

__device__ __forceinline__ uint32_t sgn_key(int v) { return (uint32_t)v ^ 0x80000000u; }
__device__ __forceinline__ int sgn_unkey(uint32_t k) { return (int)(k ^ 0x80000000u); }

// inter-CTA barrier of one frame's T co-resident CTAs (cooperative launch): a monotone counter,
// phase k waits for k*T arrivals
__device__ __forceinline__ void coop_barrier(uint32_t* ctr, uint32_t target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    uint32_t v;
    do {
      asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

// the double a sort key came from (sort_key inverse; keys of valid rows only)
__device__ __forceinline__ double key_to_double(uint64_t sk) {
  const uint64_t k = ~sk;  // score_key
  const uint64_t b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  return __longlong_as_double((long long)b);
}

template <bool BY_INDEX>
__global__ void __launch_bounds__(kCoopThreads) pnms_coop(CoopArgs ca) {
  const BinArgs& a = ca.b;
  const int T = ca.tiles;
  const int f = blockIdx.x / T, r = blockIdx.x % T;
  const long long fbase = (long long)f * a.n_max;
  const int cnt = frame_count(a.counts, f, a.n_max);
  const int W4 = ((a.W32 + 3) & ~3);
  CoopFrame* cf = ca.scr + f;
  uint32_t* mask = ca.mask + (size_t)f * W4;
  const int lane = threadIdx.x & 31;
  constexpr int NW = kCoopThreads / 32;
  // diagnostics: global timer per CTA at the phase boundaries (trace[(f*T + r)*8 + k])
#define PNMS_COOP_TRACE(k)                                                                 \
  do {                                                                                     \
    if (a.trace && threadIdx.x == 0) {                                                     \
      unsigned long long t_;                                                               \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                               \
      a.trace[((long long)f * T + r) * 8 + (k)] = t_;                                      \
    }                                                                                      \
  } while (0)
  PNMS_COOP_TRACE(0);

  __shared__ __align__(16) RecBin recS[kCoopCap];
  __shared__ __align__(16) uint4 ent[kCoopCap];          // region entries
  __shared__ __align__(16) uint64_t keyR[kCoopCap];      // keys at the cell positions
  __shared__ __align__(16) uint16_t comb[kCoopCells + 8];  // cell counts -> starts
  __shared__ uint32_t Tz[128];
  __shared__ uint32_t rowhist[kB2RowClasses];
  __shared__ uint32_t scan_tmp[64];
  __shared__ uint32_t red[16][NW];
  uint32_t* lcnt = reinterpret_cast<uint32_t*>(keyR);     // phase 1 (keyR is phase 2's): per-tile counts ...
  uint32_t* gbase = lcnt + kCoopMaxTiles;                  // ... and reserved list offsets

  if (threadIdx.x < 128) {
    const int zv = threadIdx.x;
    const uint32_t T_ = zv == 0 ? 0u : (uint32_t)ceil(ref_threshold(a.theta, zv));
    Tz[zv] = T_ | (((T_ + zv) / (uint32_t)(zv + 1)) << 16);
  }
  if (threadIdx.x < kB2RowClasses) rowhist[threadIdx.x] = 0u;
  __syncthreads();

  // ---- phase 0: this CTA's slice (kept in `ent` as list entries for phase 1; NaN rows get
  // z = 0x7F, never a valid narrow7 side); statistics; NaN rows are survivors
  const int slice = (cnt + T - 1) / T;
  const int s0 = r * slice, s1 = min(cnt, s0 + slice);
  const bool pad_rule = a.d_max > cnt;
  {
    uint32_t v[12] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};  // CoopFrame field order
    for (int e = s0 + (int)threadIdx.x; e < s1; e += kCoopThreads) {
      const long long g = fbase + e;
      const int32_t xv = a.x[g], yv = a.y[g], zv = a.z[g];
      const double sv = a.s[g];
      v[0] = max(v[0], (uint32_t)frame_mode_of(xv, yv, zv));
      {
        const uint64_t key = sort_key(sv);
        uint4 en;
        en.x = ((uint32_t)xv & 0xFFFFu) | ((uint32_t)yv << 16);
        en.y = (sv == sv ? ((uint32_t)zv & 0x7Fu) : 0x7Fu) | ((pad_rule && sv < 0.0) ? 0x80u : 0u) | ((uint32_t)e << 16);
        en.z = (uint32_t)key; en.w = (uint32_t)(key >> 32);
        ent[e - s0] = en;
      }
      if (sv == sv) {
        v[1] = max(v[1], ~sgn_key(zv)); v[2] = max(v[2], sgn_key(zv));
        v[3] = max(v[3], ~sgn_key(xv)); v[4] = max(v[4], ~sgn_key(yv));
        v[5] = max(v[5], sgn_key(xv)); v[6] = max(v[6], sgn_key(yv));
        v[7] += 1u;
        const uint32_t tw = Tz[zv & 127];
        v[8] = max(v[8], sgn_key(zv + 1 - (int)(tw >> 16)));
        v[9] = max(v[9], ~sgn_key((int)(tw >> 16)));
      } else {
        atomicOr(&mask[e >> 5], 1u << (e & 31));
      }
    }
#pragma unroll
    for (int i = 0; i < 12; ++i) {
      const uint32_t w = i == 7 ? __reduce_add_sync(0xFFFFFFFFu, v[i]) : __reduce_max_sync(0xFFFFFFFFu, v[i]);
      if (lane == 0) red[i][threadIdx.x >> 5] = w;
    }
    __syncthreads();
    if (threadIdx.x < 12) {
      const int i = threadIdx.x;
      uint32_t w = 0u;
      for (int k = 0; k < NW; ++k) w = i == 7 ? w + red[i][k] : max(w, red[i][k]);
      uint32_t* fld = reinterpret_cast<uint32_t*>(cf) + i;
      if (i == 7) { if (w) atomicAdd(fld, w); }
      else if (w) atomicMax(fld, w);
    }
  }
  PNMS_COOP_TRACE(1);
  coop_barrier(&cf->barrier, (uint32_t)T);
  PNMS_COOP_TRACE(2);

  // ---- phase 1: parameters (identical in every CTA) and the tile lists
  // the 12 accumulated fields in one L2 round trip (three 16 B loads), shared by the CTA
  __shared__ __align__(16) uint32_t hdr[16];
  if (threadIdx.x < 3) reinterpret_cast<uint4*>(hdr)[threadIdx.x] = __ldcg(reinterpret_cast<const uint4*>(cf) + threadIdx.x);
  __syncthreads();
  const CoopFrame* vf = reinterpret_cast<const CoopFrame*>(hdr);
  const int n_act = (int)vf->n_act;
  const int minz = sgn_unkey(~vf->nminz), maxz = sgn_unkey(vf->maxz);
  const bool eligible = vf->mode == (uint32_t)kNarrow7 && (n_act == 0 || (a.theta > 0.0 && minz >= 1));
  const int L = n_act ? sgn_unkey(vf->maxL) : 0, R = n_act ? sgn_unkey(~vf->nminW) : 1;
  const int ox = sgn_unkey(~vf->nminx), oy = sgn_unkey(~vf->nminy);
  const int spanx = sgn_unkey(vf->maxx) - ox, spany = sgn_unkey(vf->maxy) - oy;
  // cells as pnms_binned2.cuh: Sy = the power of two nearest L + 1, Sx = Sy / 4
  int Sy, Sx;
  {
    const int h = L + 1;
    const int p2 = 1 << (31 - __clz(h));
    Sy = (long long)h * h > 2LL * p2 * p2 ? 2 * p2 : p2;
    Sx = max(Sy >> 2, kMinCellSide);
    Sy = max(Sy, kMinCellSide);
  }
  const int shx = 31 - __clz(Sx), shy = 31 - __clz(Sy);
  const int GX = n_act ? (spanx >> shx) + 1 : 1, GY = n_act ? (spany >> shy) + 1 : 1;
  // halos: a row reaches L pixels left / up and z + 1 - R right / down
  const int hL = (L + Sx - 1) >> shx, hR = (maxz + 1 - R + Sx - 1) >> shx;
  const int vL = (L + Sy - 1) >> shy, vR = (maxz + 1 - R + Sy - 1) >> shy;
  // tile layout: TX x TY <= T tiles, square-ish in pixels
  int TX = (int)sqrtf((float)T * (float)(GX << shx) / (float)(GY << shy) + 0.5f);
  TX = max(1, min(TX, min(GX, T)));
  int TY = max(1, min(GY, T / TX));
  const int tw = (GX + TX - 1) / TX, th = (GY + TY - 1) / TY;
  TX = (GX + tw - 1) / tw;
  TY = (GY + th - 1) / th;
  const int cap = ca.cap;
  uint4* lists = ca.lists + (size_t)f * T * cap;
  if (eligible && n_act > 0) {
    // every (box, tile) pair of the slice, visited twice: first counted per tile in shared
    // memory, then written at a slot of the range one global atomic per (CTA, tile) reserved
    auto for_each_tile = [&](auto&& visit) {
      for (int q = (int)threadIdx.x; q < s1 - s0; q += kCoopThreads) {
        const uint4 en = ent[q];
        if ((en.y & 0x7Fu) == 0x7Fu) continue;  // NaN row: no cell
        const int xv = (int)(en.x & 0xFFFFu), yv = (int)(en.x >> 16);
        const int cx = (xv - ox) >> shx, cy = (yv - oy) >> shy;
        // tiles whose region [t*tw - hL, t*tw + tw - 1 + hR] holds cx (same in y);
        // ceil((c - h - tw + 1) / tw) = floor((c - h) / tw) for c >= h
        const int tx0 = max(cx - hR, 0) / tw, tx1 = min(TX - 1, (cx + hL) / tw);
        const int ty0 = max(cy - vR, 0) / th, ty1 = min(TY - 1, (cy + vL) / th);
        for (int ty = ty0; ty <= ty1; ++ty) {
          if (cy < ty * th - vL || cy > ty * th + th - 1 + vR) continue;
          for (int tx = tx0; tx <= tx1; ++tx) {
            if (cx < tx * tw - hL || cx > tx * tw + tw - 1 + hR) continue;
            visit(ty * TX + tx, en);
          }
        }
      }
    };
    for (int t = threadIdx.x; t < kCoopMaxTiles; t += kCoopThreads) lcnt[t] = 0u;
    __syncthreads();
    for_each_tile([&](int t, const uint4&) { atomicAdd(&lcnt[t], 1u); });
    __syncthreads();
    for (int t = threadIdx.x; t < TX * TY; t += kCoopThreads) {
      const uint32_t c = lcnt[t];
      gbase[t] = c ? atomicAdd(&cf->tile_cnt[t], c) : 0u;
      lcnt[t] = 0u;
    }
    __syncthreads();
    for_each_tile([&](int t, const uint4& en) {
      const uint32_t slot = gbase[t] + atomicAdd(&lcnt[t], 1u);
      if (slot < (uint32_t)cap) lists[(size_t)t * cap + slot] = en;
      else atomicOr(&cf->overflow, 1u);
    });
  }
  PNMS_COOP_TRACE(3);
  coop_barrier(&cf->barrier, 2u * T);
  PNMS_COOP_TRACE(4);

  // ---- phase 2: tile r
  if (threadIdx.x == 0) { hdr[12] = __ldcg(&cf->overflow); hdr[13] = __ldcg(&cf->tile_cnt[min(r, kCoopMaxTiles - 1)]); }
  __syncthreads();
  const bool go = eligible && n_act > 0 && hdr[12] == 0u && r < TX * TY;
  if (go) {
    const int tx = r % TX, ty = r / TX;
    const int cx0 = max(tx * tw - hL, 0), cx1 = min(tx * tw + tw - 1 + hR, GX - 1);   // region
    const int cy0 = max(ty * th - vL, 0), cy1 = min(ty * th + th - 1 + vR, GY - 1);
    const int ix0 = tx * tw, ix1 = min(tx * tw + tw, GX) - 1;                         // interior
    const int iy0 = ty * th, iy1 = min(ty * th + th, GY) - 1;
    // the region's own cell grid: the global cells, coarsened (any side is exact) until it
    // fits kCoopCells
    const int px0 = ox + (cx0 << shx), py0 = oy + (cy0 << shy);
    const int pw = (cx1 - cx0 + 1) << shx, ph = (cy1 - cy0 + 1) << shy;
    int lsx = shx, lsy = shy;
    while ((long long)(((pw - 1) >> lsx) + 1) * (((ph - 1) >> lsy) + 1) + 1 > kCoopCells) {
      if ((pw >> lsx) >= (ph >> lsy)) ++lsx;
      else ++lsy;
    }
    const int LW = ((pw - 1) >> lsx) + 1, LH = ((ph - 1) >> lsy) + 1, lcells = LW * LH;
    const int m = (int)min(hdr[13], (uint32_t)cap);
    if (lcells + 1 > kCoopCells || m > kCoopCap) {
      if (threadIdx.x == 0) atomicOr(&cf->overflow, 2u);
    } else {
      // the region's entries: cells by counting sort (no score order: the scan gates on the
      // full 64-bit keys, with the input slot for by_index ties), 16 B records + keys at the
      // cell positions, then every interior row against its window
      for (int w = threadIdx.x; w < (kCoopCells + 8) / 8; w += kCoopThreads)
        reinterpret_cast<uint4*>(comb)[w] = make_uint4(0u, 0u, 0u, 0u);
      const uint4* lst = lists + (size_t)r * cap;
      for (int q = threadIdx.x; q < m; q += kCoopThreads) ent[q] = lst[q];
      __syncthreads();
      constexpr int PE = kCoopCap / kCoopThreads;
      uint32_t cr[PE];  // local cell | rank in cell << 16
#pragma unroll
      for (int k = 0; k < PE; ++k) {
        const int q = threadIdx.x + k * kCoopThreads;
        cr[k] = 0xFFFFFFFFu;
        if (q < m) {
          const uint4 en = ent[q];
          const int xv = (int)(en.x & 0xFFFFu), yv = (int)(en.x >> 16);
          const int lc = ((yv - py0) >> lsy) * LW + ((xv - px0) >> lsx);
          cr[k] = (uint32_t)lc | (atomic_inc_u16(comb, lc) << 16);
        }
      }
      __syncthreads();
      {
        // exclusive scan of the cell counts (+ the sentinel m)
        const int len = lcells + 1;
        constexpr int PS = (kCoopCells + kCoopThreads - 1) / kCoopThreads;
        const int c0 = threadIdx.x * PS;
        uint32_t sum = 0;
        for (int t = 0; t < PS; ++t) if (c0 + t < len) sum += comb[c0 + t];
        uint32_t run = block_exclusive_scan(sum, scan_tmp, nullptr);
        for (int t = 0; t < PS; ++t) {
          const int c = c0 + t;
          if (c < len) { const uint32_t v = comb[c]; comb[c] = (uint16_t)run; run += v; }
        }
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < PE; ++k) {
        const int q = threadIdx.x + k * kCoopThreads;
        if (q < m) {
          const uint4 en = ent[q];
          const int xv = (int)(en.x & 0xFFFFu), yv = (int)(en.x >> 16), zv = (int)(en.y & 0x7Fu);
          const int pos = (int)comb[cr[k] & 0xFFFFu] + (int)(cr[k] >> 16);
          const uint32_t Tv = Tz[zv] & 0xFFFFu;
          RecBin rb;
          rb.a = ((uint32_t)(xv + zv + 1) & 0xFFFFu) | ((uint32_t)(yv + zv + 1) << 16);
          rb.nb = ((uint32_t)(-xv) & 0xFFFFu) | ((uint32_t)(-yv) << 16);
          rb.w = -(int32_t)(Tv << 17) | (zv + 1);
          rb.k = en.y >> 16;  // input slot
          recS[pos] = rb;
          keyR[pos] = ((uint64_t)en.w << 32) | en.z;
        }
      }
      __syncthreads();
      auto window = [&](int xv, int yv, int zv, int& wx0, int& wx1, int& wy0, int& wy1) {
        wx0 = max((xv - L - px0) >> lsx, 0);
        wx1 = min((xv + zv + 1 - R - px0) >> lsx, LW - 1);
        wy0 = max((yv - L - py0) >> lsy, 0);
        wy1 = min((yv + zv + 1 - R - py0) >> lsy, LH - 1);
      };
      const uint32_t rbase = static_cast<uint32_t>(__cvta_generic_to_shared(recS));
      // rows: the interior's live boxes (dead = suppressed by the padding columns)
#pragma unroll
      for (int k = 0; k < PE; ++k) {
        const int q = threadIdx.x + k * kCoopThreads;
        if (q >= m || (ent[q].y & 0x80u)) continue;
        const uint4 en = ent[q];
        const int xv = (int)(en.x & 0xFFFFu), yv = (int)(en.x >> 16), zv = (int)(en.y & 0x7Fu);
        const int gcx = (xv - ox) >> shx, gcy = (yv - oy) >> shy;
        if (gcx < ix0 || gcx > ix1 || gcy < iy0 || gcy > iy1) continue;
        const int p = (int)comb[cr[k] & 0xFFFFu] + (int)(cr[k] >> 16);
        const uint4 ri = lds128(rbase + (uint32_t)p * 16u);
        const uint64_t ki = keyR[p];
        const uint32_t zzi = __byte_perm(ri.z, 0u, 0x4040);
        int wx0, wx1, wy0, wy1;
        window(xv, yv, zv, wx0, wx1, wy0, wy1);
        bool hit = false;
        for (int yy = wy0; yy <= wy1 && !hit; ++yy) {
          int qq = comb[yy * LW + wx0];
          const int qe = comb[yy * LW + wx1 + 1];
          while (!hit && qq < qe) {
            const uint4 g = lds128(rbase + (uint32_t)qq * 16u);
            const uint64_t kj = keyR[qq];
            const uint32_t t1 = __viaddmin_s16x2(ri.x, g.y, zzi);
            const uint32_t t2 = __viaddmin_s16x2_relu(g.x, ri.y, t1);
            const uint32_t v = __vimin_s16x2_relu(t2, __byte_perm(g.z, 0u, 0x4040));
            const bool gate = kj < ki || (BY_INDEX && kj == ki && g.w < ri.w);
            hit = gate && (int)(v * v) + (int)g.z >= 0;
            ++qq;
          }
        }
        if (!hit) atomicOr(&mask[ri.w >> 5], 1u << (ri.w & 31));
      }
    }
  }
  PNMS_COOP_TRACE(5);
  coop_barrier(&cf->barrier, 3u * T);
  PNMS_COOP_TRACE(6);

  // ---- phase 3: compaction of this CTA's mask words (or the decline), then the cleanup.  One
  // L2 round trip: every thread loads its run of mask words (and thread 0 the overflow flag),
  // one block scan of their popcounts gives every word's offset; the words of this CTA's chunk
  // are published in shared memory and written out one slot per thread
  {
    constexpr int kMaxWpt = PNMS_MAX_SLOTS / 32 / kCoopThreads;
    const int W32 = a.W32;
    const int wpt = (W32 + kCoopThreads - 1) / kCoopThreads;
    const int wb = (int)threadIdx.x * wpt;
    uint32_t wv[kMaxWpt];
    uint32_t sum = 0;
#pragma unroll
    for (int i = 0; i < kMaxWpt; ++i) {
      wv[i] = (i < wpt && wb + i < W32) ? __ldcg(&mask[wb + i]) : 0u;
      sum += __popc(wv[i]);
    }
    if (threadIdx.x == 0) hdr[12] = __ldcg(&cf->overflow);
    uint32_t total;
    uint32_t off = block_exclusive_scan(sum, scan_tmp, &total);  // (its barriers publish hdr[12])
    const bool declined = !eligible || (n_act > 0 && hdr[12] != 0u);
    if (declined) {
      if (r == 0 && threadIdx.x == 0) binned_decline(a, f);
    } else {
      __shared__ uint32_t s_cw[64], s_co[64];
      const int wpc = (W32 + T - 1) / T;  // <= 32: T >= n / kCoopCap (coop_tiles)
      const int w0 = min(r * wpc, W32), w1 = min(w0 + wpc, W32);
#pragma unroll
      for (int i = 0; i < kMaxWpt; ++i) {
        const int w = wb + i;
        if (i < wpt && w >= w0 && w < w1 && w - w0 < 64) { s_cw[w - w0] = wv[i]; s_co[w - w0] = off; }
        off += __popc(wv[i]);
      }
      __syncthreads();
      for (int sl = w0 * 32 + (int)threadIdx.x; sl < w1 * 32; sl += kCoopThreads) {
        const int wi = (sl >> 5) - w0;
        const uint32_t bits = s_cw[wi];
        if (((bits >> lane) & 1u) && a.keep_idx) a.keep_idx[fbase + s_co[wi] + __popc(bits & lanemask_lt())] = sl;
        if (lane == 0 && a.keep_mask) a.keep_mask[(long long)f * W32 + (sl >> 5)] = bits;
      }
      if (r == 0 && threadIdx.x == 0) {
        if (a.keep_count) a.keep_count[f] = (int32_t)total;
        a.fallback[f] = 0;
      }
    }
  }
  // the last CTA of the frame re-zeroes its scratch (every CTA has read the mask by now)
  __syncthreads();
  __shared__ uint32_t s_last;
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&cf->done, 1u) == (uint32_t)T - 1;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    uint32_t* z32 = reinterpret_cast<uint32_t*>(cf);
    for (int i = threadIdx.x; i < (int)(sizeof(CoopFrame) / 4); i += kCoopThreads) z32[i] = 0u;
    for (int w = threadIdx.x; w < W4; w += kCoopThreads) mask[w] = 0u;
  }
  PNMS_COOP_TRACE(7);
#undef PNMS_COOP_TRACE
}

}  // namespace pnms

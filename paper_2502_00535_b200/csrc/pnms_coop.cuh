// pnms_coop.cuh — latency path for single large frames: one cooperative launch of T CTAs per
// frame (all co-resident) that share the frame-level work through global memory instead of
// repeating it in every CTA (pnms_binned_tiles.cuh streams the whole frame into each of its
// 128 CTAs twice).
//
//   phase 0  CTA r reads its slice of the frame once: statistics into the frame's global
//            accumulators (shared-memory reduction, one atomic per field per CTA)
//   barrier
//   phase 1  every CTA derives the same parameters (eligibility, the theta reach L / R of
//            pnms_binned2.cuh, cells, a tile layout of T tiles with halos covering the reach)
//            and appends each box of its slice to the list of every tile whose region (tile
//            plus halo) holds the box's cell: one 16 B entry {x|y<<16, z|dead<<7|slot<<16, key};
//            NaN rows of the slice are survivors (their mask bits)
//   barrier
//   phase 2  CTA r owns tile r: its region's entries into shared memory (the first 256 loaded
//            with the list's count), a counting sort into the region's cells, 16 B records
//            plus the 64-bit keys at the cell positions, and the rows of the tile's interior
//            scanned against their windows with the reference's gate on the full keys
//            (engine.py:233-235; the input slot breaks by_index ties); survivor bits into the
//            frame's global mask
//   barrier
//   phase 3  CTA r compacts mask words [r*wpc, (r+1)*wpc) into ascending keep indices (its
//            offset = popcount of the words before it), then clears the scratch the next call
//            needs zero (stores only: no cleanup round trip, see CoopFrame)
//
// Exactness is that of pnms_binned2.cuh: every column that can clear row i's bit lies in i's
// window, the window of an interior row lies inside the tile's region, and the gate compares
// the frame's own 64-bit keys.  A frame the culling cannot take (not narrow7, a T = 0 column,
// a tile region over kCoopCap boxes or kCoopCells cells) is finished inside the kernel by an
// exact O(n^2 / T)-per-CTA pass after barrier 3 (coop_exact_slice) and one more barrier — no
// dispatcher or fallback chain runs behind the kernel, which is what a call of this path
// costs on the device: the one launch.
#pragma once
#include "../../include/parnms_b200.h"
#include "pnms_binned2.cuh"

namespace pnms {

constexpr int kCoopThreads = 256;
constexpr int kCoopCap = 1024;          // region entries a tile CTA holds
constexpr int kCoopCells = 2048;        // region cells a tile CTA holds
constexpr int kCoopMaxFrames = 2;       // frames per call (latency path)
constexpr int kCoopMaxTiles = 512;
constexpr int kCoopBoxesPerTile = 128;  // default tile count: one tile per this many slots
// items per step of a row's walk (measured: 2 and 4 alike, 1 slower; more threads per row
// slower — the per-row setup, not the candidate loop, sets the walk's time)
constexpr int kCoopUnroll = 2;
constexpr int kCoopSpecLoad = 256;  // list entries loaded with the tile's count

constexpr int kCoopMaskWords = PNMS_MAX_SLOTS / 32;  // survivor words of one frame

// per-frame scratch in the caller's persistent zeroed workspace head (zero before the first
// call).  No call ends with a cleanup round trip: the barrier counters are monotone (a call's
// parity is bit 0 of its index, coop_barrier); the statistics (read by every CTA in phase 1) and
// each tile's list count (read by its own CTA in phase 2) are re-zeroed with plain stores at the
// end of the call, and the survivor mask and overflow flag are double-buffered by call parity
// (a call zeroes the other parity's, which the previous call used).  Every statistics field's
// identity is 0 (minima are kept as maxima of complements).
struct CoopFrame {
  uint32_t mode, nminz, maxz, nminx, nminy, maxx, maxy, n_act;  // ox(v) = v ^ 2^31: signed order
  uint32_t maxL, nminW, pad0, pad1;
  unsigned long long bar;  // barrier arrivals, kCoopCallStride per call (coop_barrier)
  unsigned long long bar4; // arrivals at the fourth barrier (declined frames only), T per such call
  uint32_t overflow[2];    // by call parity
  uint32_t pad2[2];
  uint32_t tile_cnt[kCoopMaxTiles];
};
static_assert(sizeof(CoopFrame) % 16 == 0, "CoopFrame layout");
// frame scratch + survivor masks ([frame][parity][kCoopMaskWords])
constexpr size_t kCoopScratchBytes = (size_t)kCoopMaxFrames * (sizeof(CoopFrame) + 2 * kCoopMaskWords * 4);

struct CoopArgs {
  BinArgs b;
  CoopFrame* scr;      // [kCoopMaxFrames] frame scratch (CoopFrame: valid between calls)
  uint32_t* mask;      // [kCoopMaxFrames][2][kCoopMaskWords] survivor bits by call parity
  uint4* lists;        // [batch][T][cap] tile entries
  int tiles;           // T: CTAs per frame
  int cap;             // entries per tile list
  int count_fallback;  // count the frames finished by coop_exact_slice in b.decl_count
};

__device__ __forceinline__ uint32_t sgn_key(int v) { return (uint32_t)v ^ 0x80000000u; }
__device__ __forceinline__ int sgn_unkey(uint32_t k) { return (int)(k ^ 0x80000000u); }

// inter-CTA barrier of one frame's T co-resident CTAs (cooperative launch) on a monotone 64-bit
// counter that is never reset: every call adds exactly kCoopCallStride to it (one arrival per
// CTA at each of the three barriers, CTA 0 adding the remainder at the third), so a call's base
// is the counter at its start rounded down to kCoopCallStride (before barrier 1 completes at
// most T - 1 < kCoopCallStride arrivals of the call are in it); barrier b waits for base + b*T,
// the third for base + kCoopCallStride
constexpr unsigned long long kCoopCallStride = 4096;
static_assert(3 * kCoopMaxTiles < kCoopCallStride, "call stride");
__device__ __forceinline__ void coop_barrier(unsigned long long* bar, unsigned long long add,
                                             unsigned long long target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    // release: the CTA's writes (ordered before thread 0 by the CTA barrier) become visible
    // to every CTA that acquires the count
    asm volatile("red.release.gpu.global.add.u64 [%0], %1;" :: "l"(bar), "l"(add) : "memory");
    unsigned long long v;
    do {
      __nanosleep(32);  // fewer polls on the line the arrivals update (measured 0.1-0.4 us per call)
      asm volatile("ld.acquire.gpu.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory");
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

// A frame the culling cannot take, finished inside the kernel: the rows of this CTA's slice
// [s0, s1) against every column of the frame in chunks of kCoopThreads, with the reference's
// own int32-wrap / float64 pair test (suppress_wide, engine.py:194-235) and the gate on the
// 64-bit keys (the input slot for by_index ties): O(n^2 / T) per CTA — the path's exact
// fallback for frames outside narrow7, with a T = 0 column or an overflowing tile.  Survivor
// bits of the slice are rewritten in `mask`.  Shared memory (the kernel's, free in phase 3):
// sA 16 KB (column records, row keys), sB 16 KB (row geometry), sK 8 KB (column keys, row state).
template <bool BY_INDEX>
__device__ __forceinline__ void coop_exact_slice(const BinArgs& a, int f, int s0, int s1, bool pad_rule, uint32_t* mask,
                                              uint32_t* sA, uint32_t* sB, uint64_t* sK) {
  static_assert(kCoopThreads * sizeof(RecWide) + kCoopCap * 8 <= kCoopCap * sizeof(RecBin), "sA");
  static_assert(kCoopThreads * 8 + kCoopCap * 4 <= kCoopCap * 8, "sK");
  RecWide* col = reinterpret_cast<RecWide*>(sA);                            // [kCoopThreads]
  uint64_t* rkey = reinterpret_cast<uint64_t*>(sA) + kCoopThreads * sizeof(RecWide) / 8;  // [kCoopCap]
  int4* rgeo = reinterpret_cast<int4*>(sB);                                 // [kCoopCap]
  uint64_t* ckey = sK;                                                      // [kCoopThreads]
  uint32_t* rst = reinterpret_cast<uint32_t*>(sK + kCoopThreads);           // [kCoopCap] 0 test, 1 out, 2 NaN
  const long long fbase = (long long)f * a.n_max;
  const int cnt = frame_count(a.counts, f, a.n_max);
  const int m = s1 - s0;
  __syncthreads();
  for (int o = threadIdx.x; o < m; o += kCoopThreads) {
    const long long g = fbase + s0 + o;
    const double sv = a.s[g];
    const RecWide w = make_rec_wide(a.x[g], a.y[g], a.z[g], a.theta);
    rgeo[o] = make_int4(w.x, w.y, w.xe, w.ye);
    rkey[o] = sort_key(sv);
    rst[o] = sv != sv ? 2u : (pad_rule && sv < 0.0) ? 1u : 0u;  // NaN never gated; padding rule
  }
  // G threads per row (a power of two, as the slice allows), thread g of a row tests columns
  // g, g + G, ... of every chunk; at most 4 rows per thread (m <= kCoopCap)
  const int G = m <= kCoopThreads / 8 ? 8 : m <= kCoopThreads / 4 ? 4 : m <= kCoopThreads / 2 ? 2 : 1;
  const int g = (int)threadIdx.x & (G - 1), o0 = (int)threadIdx.x / G, ostep = kCoopThreads / G;
  uint32_t hits = 0;  // bit k: row o0 + k * ostep is suppressed
  for (int c0 = 0; c0 < cnt; c0 += kCoopThreads) {
    __syncthreads();
    const int j = c0 + (int)threadIdx.x;
    if (j < cnt) {
      const long long g2 = fbase + j;
      col[threadIdx.x] = make_rec_wide(a.x[g2], a.y[g2], a.z[g2], a.theta);
      ckey[threadIdx.x] = sort_key(a.s[g2]);
    }
    __syncthreads();
    const int clen = min(kCoopThreads, cnt - c0);
    int k = 0;
    for (int o = o0; o < m; o += ostep, ++k) {
      if (rst[o] != 0u || ((hits >> k) & 1u)) continue;
      const int4 rg = rgeo[o];
      RecWide ri;
      ri.x = rg.x; ri.y = rg.y; ri.xe = rg.z; ri.ye = rg.w;
      const uint64_t ki = rkey[o];
      const int i = s0 + o;
      bool hit = false;
      for (int c = g; c < clen && !hit; c += G) {
        const uint64_t kj = ckey[c];
        const bool gate = kj < ki || (BY_INDEX && kj == ki && c0 + c < i);
        hit = gate && suppress_wide(ri, col[c]);
      }
      if (hit) hits |= 1u << k;
    }
  }
  __syncthreads();
  {
    int k = 0;
    for (int o = o0; o < m; o += ostep, ++k)
      if ((hits >> k) & 1u) atomicOr(&rst[o], 1u);
  }
  __syncthreads();
  for (int o = threadIdx.x; o < m; o += kCoopThreads) {
    const int i = s0 + o;
    const uint32_t bit = 1u << (i & 31);
    if (rst[o] & 1u) atomicAnd(&mask[i >> 5], ~bit);
    else atomicOr(&mask[i >> 5], bit);
  }
}

template <bool BY_INDEX>
__global__ void __launch_bounds__(kCoopThreads) pnms_coop(CoopArgs ca) {
  const BinArgs& a = ca.b;
  const int T = ca.tiles;
  const int f = blockIdx.x / T, r = blockIdx.x % T;
  const long long fbase = (long long)f * a.n_max;
  const int cnt = frame_count(a.counts, f, a.n_max);
  CoopFrame* cf = ca.scr + f;
  const int lane = threadIdx.x & 31;
  constexpr int NW = kCoopThreads / 32;
  // diagnostics: global timer per CTA at the phase boundaries (trace[(f*T + r)*24 + k]; k = 8..15 inside phases 1 and 2, 16: SM id + 1)
#define PNMS_COOP_TRACE(k)                                                                 \
  do {                                                                                     \
    if (a.trace && threadIdx.x == 0) {                                                     \
      unsigned long long t_;                                                               \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                               \
      a.trace[((long long)f * T + r) * 24 + (k)] = t_;                                      \
    }                                                                                      \
  } while (0)
  PNMS_COOP_TRACE(0);
  pdl_trigger();  // the fallback dispatcher may launch early (PDL; it waits for this grid)
  if (a.trace && threadIdx.x == 0) {
    uint32_t smid_;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid_));
    a.trace[((long long)f * T + r) * 24 + 16] = smid_ + 1;
  }

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
  // this call's barrier base and parity (coop_barrier), loaded under phase 0
  __shared__ unsigned long long s_base, s_base4;
  ulonglong2 bar0 = make_ulonglong2(0ull, 0ull);
  if (threadIdx.x == 0) bar0 = __ldcg(reinterpret_cast<const ulonglong2*>(&cf->bar));

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
      }
    }
    if (threadIdx.x == 0) {
      s_base = bar0.x & ~(kCoopCallStride - 1);
      s_base4 = bar0.y;  // exact: no CTA passes barrier 3 before this one reaches barrier 1
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
  const unsigned long long bbase = s_base;
  const int par = (int)(bbase / kCoopCallStride) & 1;
  uint32_t* mask = ca.mask + ((size_t)f * 2 + par) * kCoopMaskWords;
  PNMS_COOP_TRACE(1);
  coop_barrier(&cf->bar, 1ull, bbase + (unsigned long long)T);
  PNMS_COOP_TRACE(2);
  // NaN rows of the slice survive (their mask bits)
  for (int q = (int)threadIdx.x; q < s1 - s0; q += kCoopThreads)
    if ((ent[q].y & 0x7Fu) == 0x7Fu) atomicOr(&mask[(s0 + q) >> 5], 1u << ((s0 + q) & 31));

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
    PNMS_COOP_TRACE(12);
    for_each_tile([&](int t, const uint4&) { atomicAdd(&lcnt[t], 1u); });
    __syncthreads();
    for (int t = threadIdx.x; t < TX * TY; t += kCoopThreads) {
      const uint32_t c = lcnt[t];
      gbase[t] = c ? atomicAdd(&cf->tile_cnt[t], c) : 0u;
      lcnt[t] = 0u;
    }
    __syncthreads();
    PNMS_COOP_TRACE(13);
    for_each_tile([&](int t, const uint4& en) {
      const uint32_t slot = gbase[t] + atomicAdd(&lcnt[t], 1u);
      if (slot < (uint32_t)cap) lists[(size_t)t * cap + slot] = en;
      else atomicOr(&cf->overflow[par], 1u);
    });
  }
  PNMS_COOP_TRACE(3);
  coop_barrier(&cf->bar, 1ull, bbase + 2ull * (unsigned long long)T);
  PNMS_COOP_TRACE(4);

  // ---- phase 2: tile r
  if (threadIdx.x == 0) {
    hdr[12] = __ldcg(&cf->overflow[par]);
    hdr[13] = __ldcg(&cf->tile_cnt[min(r, kCoopMaxTiles - 1)]);
  }
  // the first kCoopSpecLoad entries of this tile's list are loaded with its count (one L2 round
  // trip; entries past the count are in the list's allocation and ignored)
  const uint4* lst = ca.lists + ((size_t)f * T + (size_t)min(r, T - 1)) * ca.cap;
  uint4 spec[kCoopSpecLoad / kCoopThreads + 1];
#pragma unroll
  for (int k = 0; k < kCoopSpecLoad / kCoopThreads; ++k) spec[k] = __ldcg(lst + threadIdx.x + k * kCoopThreads);
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
      if (threadIdx.x == 0) atomicOr(&cf->overflow[par], 2u);
    } else {
      // the region's entries: cells by counting sort (no score order: the scan gates on the
      // full 64-bit keys, with the input slot for by_index ties), 16 B records + keys at the
      // cell positions, then every interior row against its window
      for (int w = threadIdx.x; w < (kCoopCells + 8) / 8; w += kCoopThreads)
        reinterpret_cast<uint4*>(comb)[w] = make_uint4(0u, 0u, 0u, 0u);
      for (int q = threadIdx.x + kCoopSpecLoad; q < m; q += kCoopThreads) ent[q] = lst[q];
#pragma unroll
      for (int k = 0; k < kCoopSpecLoad / kCoopThreads; ++k) {
        const int q = threadIdx.x + k * kCoopThreads;
        if (q < m) ent[q] = spec[k];
      }
      __syncthreads();
      PNMS_COOP_TRACE(8);
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
      PNMS_COOP_TRACE(9);
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
      PNMS_COOP_TRACE(10);
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
          // a row: a live box of the interior (dead = suppressed by the padding columns)
          const int gcx = (xv - ox) >> shx, gcy = (yv - oy) >> shy;
          const bool row = !(en.y & 0x80u) && gcx >= ix0 && gcx <= ix1 && gcy >= iy0 && gcy <= iy1;
          cr[k] = row ? (uint32_t)pos : 0xFFFFFFFFu;
        } else {
          cr[k] = 0xFFFFFFFFu;
        }
      }
      if (threadIdx.x == 0) rowhist[0] = 0u;
      __syncthreads();
      PNMS_COOP_TRACE(11);
      // the row list (record positions) and per-row hit flags, in `ent` (read out above)
      uint16_t* rows = reinterpret_cast<uint16_t*>(ent);
      uint32_t* hf = reinterpret_cast<uint32_t*>(ent) + kCoopCap / 2;
#pragma unroll
      for (int k = 0; k < PE; ++k) {
        const bool row = cr[k] != 0xFFFFFFFFu;
        const uint32_t bal = __ballot_sync(0xFFFFFFFFu, row);
        uint32_t base = 0;
        if (lane == 0 && bal) base = atomicAdd(&rowhist[0], (uint32_t)__popc(bal));
        base = __shfl_sync(0xFFFFFFFFu, base, 0);
        if (row) {
          const uint32_t slot = base + __popc(bal & lanemask_lt());
          rows[slot] = (uint16_t)cr[k];
          hf[slot] = 0u;
        }
      }
      __syncthreads();
      PNMS_COOP_TRACE(14);
      // every row against its window's records, gate on the full 64-bit keys (the input slot
      // breaks by_index ties).  The scan is latency-bound (a tile's time is its longest row), so
      // G threads share a row (G = 8 .. 2 as the rows allow: item k of the row's cell runs,
      // walked as one sequence, is thread k mod G's) and a thread tests 4 items per step
      // (independent loads; an index past the run's end is clamped to its last record — an
      // extra test of a window record cannot change the row's outcome)
      const int nr = (int)rowhist[0];
            const int G = nr <= kCoopThreads / 8 ? 8 : nr <= kCoopThreads / 4 ? 4 : nr <= kCoopThreads / 2 ? 2 : 1;
      const int g = (int)threadIdx.x & (G - 1);
      const uint32_t rbase = static_cast<uint32_t>(__cvta_generic_to_shared(recS));
      for (int o = (int)threadIdx.x / G; o < nr; o += kCoopThreads / G) {
        const int p = rows[o];
        const uint4 ri = lds128(rbase + (uint32_t)p * 16u);
        const uint64_t ki = keyR[p];
        const uint32_t zzi = __byte_perm(ri.z, 0u, 0x4040);
        const int xv = -(int)(int16_t)(ri.y & 0xFFFFu), yv = -(int)(int16_t)(ri.y >> 16);
        const int zv = (int)(ri.z & 0xFFu) - 1;
        const int wx0 = max((xv - L - px0) >> lsx, 0), wx1 = min((xv + zv + 1 - R - px0) >> lsx, LW - 1);
        const int wy0 = max((yv - L - py0) >> lsy, 0), wy1 = min((yv + zv + 1 - R - py0) >> lsy, LH - 1);
        auto test = [&](int q) {
          const uint4 gj = lds128(rbase + (uint32_t)q * 16u);
          const uint64_t kj = keyR[q];
          const uint32_t t1 = __viaddmin_s16x2(ri.x, gj.y, zzi);
          const uint32_t t2 = __viaddmin_s16x2_relu(gj.x, ri.y, t1);
          const uint32_t v = __vimin_s16x2_relu(t2, __byte_perm(gj.z, 0u, 0x4040));
          const bool gate = kj < ki || (BY_INDEX && kj == ki && gj.w < ri.w);
          return gate && (int)(v * v) + (int)gj.z >= 0;
        };
        bool hit = false;
        int B = 0;  // items of the row's runs before this one
        for (int yy = wy0; yy <= wy1 && !hit; ++yy) {
          const int qb = comb[yy * LW + wx0], qe = comb[yy * LW + wx1 + 1];
          for (int qq = qb + ((g - B) & (G - 1)); !hit && qq < qe; qq += kCoopUnroll * G) {
            bool h = test(qq);
#pragma unroll
            for (int u = 1; u < kCoopUnroll; ++u) h |= test(min(qq + u * G, qe - 1));
            hit = h;
          }
          B += qe - qb;
        }
        if (hit) atomicOr(&hf[o], 1u);
      }
      __syncthreads();
      PNMS_COOP_TRACE(15);
      for (int o = threadIdx.x; o < nr; o += kCoopThreads) {
        if (!hf[o]) {
          const uint32_t sl = recS[rows[o]].k;
          atomicOr(&mask[sl >> 5], 1u << (sl & 31));
        }
      }
    }
  }
  PNMS_COOP_TRACE(5);
  coop_barrier(&cf->bar, r == 0 ? 1ull + kCoopCallStride - 3ull * (unsigned long long)T : 1ull, bbase + kCoopCallStride);
  PNMS_COOP_TRACE(6);

  // ---- phase 3: compaction of this CTA's mask words.  One L2 round trip: every thread loads
  // its run of mask words (and thread 0 the overflow flag), one block scan of their popcounts
  // gives every word's offset; the words of this CTA's chunk are published in shared memory and
  // written out one slot per thread.  A frame the culling cannot take (not narrow7, a T = 0
  // column, an overflowing tile) is finished here first, exactly (coop_exact_slice), so no
  // fallback chain runs behind the kernel.
  bool declined;
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
    if (threadIdx.x == 0) hdr[12] = __ldcg(&cf->overflow[par]);
    uint32_t total;
    uint32_t off = block_exclusive_scan(sum, scan_tmp, &total);  // (its barriers publish hdr[12])
    declined = !eligible || (n_act > 0 && hdr[12] != 0u);
    if (declined) {
      coop_exact_slice<BY_INDEX>(a, f, s0, s1, pad_rule, mask, reinterpret_cast<uint32_t*>(recS),
                                 reinterpret_cast<uint32_t*>(ent), keyR);
      if (ca.count_fallback && r == 0 && threadIdx.x == 0) atomicAdd(a.decl_count, 1);
      coop_barrier(&cf->bar4, 1ull, s_base4 + (unsigned long long)T);
      sum = 0;
#pragma unroll
      for (int i = 0; i < kMaxWpt; ++i) {
        wv[i] = (i < wpt && wb + i < W32) ? __ldcg(&mask[wb + i]) : 0u;
        sum += __popc(wv[i]);
      }
      off = block_exclusive_scan(sum, scan_tmp, &total);
    }
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
  // scratch for the next call (stores at the end: zeroing in phase 2 measured 4 us slower, the
  // stores stalling the list reads): the tile's count (its CTA is its only reader), the
  // statistics (read by every CTA in phase 1), the other parity's mask and overflow flag
  if (threadIdx.x == 0) cf->tile_cnt[min(r, kCoopMaxTiles - 1)] = 0u;
  if (r == 0 && threadIdx.x < 12) reinterpret_cast<uint32_t*>(cf)[threadIdx.x] = 0u;
  {
    uint32_t* omask = ca.mask + ((size_t)f * 2 + (par ^ 1)) * kCoopMaskWords;
    const int ch = (kCoopMaskWords + T - 1) / T, w1 = min((r + 1) * ch, kCoopMaskWords);
    for (int w = r * ch + (int)threadIdx.x; w < w1; w += kCoopThreads) omask[w] = 0u;
    if (r == 0 && threadIdx.x == 0) cf->overflow[par ^ 1] = 0u;
  }
  PNMS_COOP_TRACE(7);
#undef PNMS_COOP_TRACE
}

}  // namespace pnms

// pnms_binned_cluster.cuh — the exact binned NMS of pnms_binned.cuh for frames too large for
// one CTA (4096 < n <= kClMaxSlots, e.g. the 16384-box 4K frame of BASELINE config 3), run by
// one thread-block cluster of CS CTAs per frame with everything in distributed shared memory.
//
//   CTA r loads input slots [r*slice, (r+1)*slice) once (register stash) and owns
//     - the cell rows of band r: cy with floor(cy*CS/GY) == r (balanced bands), and
//     - the survivor bits of its input slice.
//   stats      block reduce -> atomics into CTA 0's shared memory (DSMEM)         cluster.sync
//   histogram  atomicAdd on the owning CTA's cell counters (the return value is the rank
//              of the box inside its cell)                                           cluster.sync
//   scan       each CTA scans its own band's cells; largest cell / capacity checks    cluster.sync
//   scatter    16 B records, keys and slots stored straight into the owner's smem     cluster.sync
//   sort       per-cell insertion sort by (key, slot) + skip distances (own cells)    cluster.sync
//   scan rows  each CTA scans its own rows; the reachable cell rows of the bands above
//              and below are read through DSMEM; survivor bits land in the slice
//              owner's words (DSMEM atomicOr)                                        cluster.sync
//   compact    per-slice popcounts -> cluster prefix -> ascending keep indices        cluster.sync
// Exactness argument, record format and eligibility are those of pnms_binned.cuh; a declined
// frame (ineligible, a cell over kBinCellMax boxes, a band over kClCap boxes) is appended to
// the declined-frame list for the dense pipeline.
#pragma once
#include <cooperative_groups.h>

#include "pnms_binned.cuh"

namespace pnms {

namespace cgc = cooperative_groups;

constexpr int kClThreads = 1024;
constexpr int kClCap = 3072;          // boxes a CTA's band may hold
constexpr int kClCells = 2048;        // cells a CTA's band may hold
constexpr int kClMaxSlice = 4096;     // input slots per CTA (register stash: 8 per thread)

struct __align__(16) ClStats {
  int mode, minz, maxz, minx, miny, maxx, maxy, big, n_act, over, maxL, minW, pad_[4];
  uint32_t total[16];                 // per-CTA survivor counts (compaction prefix)
};

inline size_t binned_cluster_smem_bytes() {
  return (size_t)kClCap * 2 * (sizeof(RecBin) + 8 + 2 + 2) + (size_t)(kClCells + 4) * 4 * 2 + (kClMaxSlice / 32 + 4) * 4 +
         64 * 4 + sizeof(ClStats) + 64;
}

// One row against the gate-passing prefixes of its reachable cells (the scan of
// pnms_binned_frame), with the cell rows' storage supplied per cell row yy: `base(yy)` is
// the first local cell index of the row, the other accessors return that row's arrays.
template <bool BY_INDEX, class Base, class CS_, class RR, class KR, class IR, class SELF>
__device__ __forceinline__ bool cluster_row_scan(const RecBin& ri, int p, int cx0, int cx1, int cy0, int cy1, Base base,
                                                 CS_ cs_of, RR rec_of, KR key_of, IR idx_of, SELF is_self,
                                                 uint64_t ki, int ii) {
  const uint32_t zzi = __byte_perm((uint32_t)ri.w, 0u, 0x4040);
  bool sup = false, tie = false;
  for (int yy = cy0; yy <= cy1 && !sup; ++yy) {
    const int lr = base(yy);
    const uint32_t* cs = cs_of(yy);
    const RecBin* rr = rec_of(yy);
    int q = (int)cs[lr + cx0];
    const int qe = (int)cs[lr + cx1 + 1];
    const int self_p = is_self(yy) ? p : -1;
    while (q < qe) {
      const RecBin g = rr[q];
      const bool gate = g.k < ri.k;
      tie |= (g.k == ri.k) & (q != self_p);
      const uint32_t t1 = __viaddmin_s16x2(ri.a, g.nb, zzi);
      const uint32_t t2 = __viaddmin_s16x2_relu(g.a, ri.nb, t1);
      const uint32_t v = __vimin_s16x2_relu(t2, __byte_perm((uint32_t)g.w, 0u, 0x4040));
      if (gate && (int)(v * v) + g.w >= 0) {
        sup = true;
        break;
      }
      q += gate ? 1 : (int)__byte_perm((uint32_t)g.w, 0u, 0x4441);
    }
  }
  if (!sup && tie) {
    // exact rescan on full keys (and slots for by_index), as pnms_binned_frame
    for (int yy = cy0; yy <= cy1 && !sup; ++yy) {
      const int lr = base(yy);
      const uint32_t* cs = cs_of(yy);
      const RecBin* rr = rec_of(yy);
      const uint64_t* kr = key_of(yy);
      const uint16_t* ir = idx_of(yy);
      int q = (int)cs[lr + cx0];
      const int qe = (int)cs[lr + cx1 + 1];
      while (q < qe) {
        const uint64_t kj = kr[q];
        const RecBin rj = rr[q];
        if (kj < ki || (BY_INDEX && kj == ki && (int)ir[q] < ii)) {
          const uint32_t t1 = __viaddmin_s16x2(ri.a, rj.nb, zzi);
          const uint32_t t2 = __viaddmin_s16x2_relu(rj.a, ri.nb, t1);
          const uint32_t v = __vimin_s16x2_relu(t2, __byte_perm((uint32_t)rj.w, 0u, 0x4040));
          if ((int)(v * v) + rj.w >= 0) {
            sup = true;
            break;
          }
          ++q;
        } else {
          q += __byte_perm((uint32_t)rj.w, 0u, 0x4441);
        }
      }
    }
  }
  return sup;
}

// diagnostics: per-CTA global timer after each cluster barrier (trace[r * 16 + phase])
#define PNMS_CL_TRACE(ph)                                                                      \
  do {                                                                                         \
    if (trace && threadIdx.x == 0) {                                                           \
      unsigned long long t_;                                                                   \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                   \
      trace[r * 16 + (ph)] = t_;                                                               \
    }                                                                                          \
  } while (0)

template <bool BY_INDEX, int CS, int PER>
__global__ void __launch_bounds__(kClThreads, 1) pnms_binned_cluster(BinArgs a, int slice) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cgc::cluster_group cl = cgc::this_cluster();
  const int r = (int)cl.block_rank();
  const int f = blockIdx.x / CS;
  const long long fbase = (long long)f * a.n_max;
  const int cnt = frame_count(a.counts, f, a.n_max);
  RecBin* recS = reinterpret_cast<RecBin*>(smem_raw);
  uint64_t* keyS = reinterpret_cast<uint64_t*>(recS + kClCap);
  uint16_t* idxS = reinterpret_cast<uint16_t*>(keyS + kClCap);
  // arrival-order staging of the scatter (cell-grouped, unsorted inside a cell)
  RecBin* tRec = reinterpret_cast<RecBin*>(idxS + 2 * kClCap);   // 2*kClCap u16 keeps 16 B alignment
  uint64_t* tKey = reinterpret_cast<uint64_t*>(tRec + kClCap);
  uint16_t* tIdx = reinterpret_cast<uint16_t*>(tKey + kClCap);
  uint16_t* tCell = tIdx + kClCap;
  uint32_t* cstart = reinterpret_cast<uint32_t*>(tCell + kClCap);
  uint32_t* ecs = cstart + kClCells + 4;        // cell starts of the halo-extended band
  uint32_t* kbits = ecs + kClCells + 4;
  uint32_t* scan_tmp = kbits + kClMaxSlice / 32 + 4;
  ClStats* st = reinterpret_cast<ClStats*>(scan_tmp + 64);
  ClStats* st0 = cl.map_shared_rank(st, 0);
  const int e0 = r * slice;
  const int slice_words = slice / 32;
  unsigned long long* trace = a.trace;  // diagnostics: phase timestamps (pnms_debug_trace)

  // T_z | wmin_z << 16 (pnms_binned2.cuh): the theta reach of a suppressing column
  __shared__ uint32_t Tz[128];
  if (threadIdx.x < 128) {
    const int zv = threadIdx.x;
    const uint32_t T = zv == 0 ? 0u : (uint32_t)ceil(ref_threshold(a.theta, zv));
    Tz[zv] = T | (((T + zv) / (uint32_t)(zv + 1)) << 16);
  }
  if (threadIdx.x == 0) {
    st->mode = kNarrow7; st->minz = 0x7FFFFFFF; st->maxz = 0;
    st->minx = st->miny = 0x7FFFFFFF; st->maxx = st->maxy = -0x7FFFFFFF;
    st->big = 0; st->n_act = 0; st->over = 0; st->maxL = 0; st->minW = 0x7FFFFFFF;
  }
  for (int w = threadIdx.x; w < slice_words; w += kClThreads) kbits[w] = 0u;
  for (int c = threadIdx.x; c < kClCells + 4; c += kClThreads) cstart[c] = 0u;
  cl.sync();
  PNMS_CL_TRACE(0);
  // ---- pass 1: own input slice, once from HBM; statistics into CTA 0
  uint32_t xy[PER], zc[PER];
  {
    int mode = kNarrow7, minz = 0x7FFFFFFF, maxz = 0, n_act = 0, maxL = 0, minW = 0x7FFFFFFF;
    int minx = 0x7FFFFFFF, miny = 0x7FFFFFFF, maxx = -0x7FFFFFFF, maxy = -0x7FFFFFFF;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int el = threadIdx.x + k * kClThreads;
      const int e = e0 + el;
      xy[k] = 0u; zc[k] = 0xFFFFFFFFu;
      if (el < slice && e < cnt) {
        const long long g = fbase + e;
        const int32_t xv = a.x[g], yv = a.y[g], zv = a.z[g];
        const double sv = a.s[g];
        mode = max(mode, frame_mode_of(xv, yv, zv));
        if (sv == sv) {
          ++n_act;
          minz = min(minz, zv); maxz = max(maxz, zv);
          minx = min(minx, xv); maxx = max(maxx, xv);
          miny = min(miny, yv); maxy = max(maxy, yv);
          const uint32_t tw = Tz[zv & 127];
          maxL = max(maxL, zv + 1 - (int)(tw >> 16)); minW = min(minW, (int)(tw >> 16));
          xy[k] = ((uint32_t)xv & 0xFFFFu) | ((uint32_t)yv << 16);
          zc[k] = (uint32_t)zv & 0xFFu;
        } else {
          atomicOr(&kbits[el >> 5], 1u << (el & 31));  // NaN: never gated, never suppresses
        }
      }
    }
    mode = __reduce_max_sync(0xFFFFFFFFu, mode);
    minz = __reduce_min_sync(0xFFFFFFFFu, minz);
    maxz = __reduce_max_sync(0xFFFFFFFFu, maxz);
    n_act = __reduce_add_sync(0xFFFFFFFFu, n_act);
    minx = __reduce_min_sync(0xFFFFFFFFu, minx); maxx = __reduce_max_sync(0xFFFFFFFFu, maxx);
    miny = __reduce_min_sync(0xFFFFFFFFu, miny); maxy = __reduce_max_sync(0xFFFFFFFFu, maxy);
    maxL = __reduce_max_sync(0xFFFFFFFFu, maxL); minW = __reduce_min_sync(0xFFFFFFFFu, minW);
    if ((threadIdx.x & 31) == 0) {
      atomicMax(&st0->maxL, maxL); atomicMin(&st0->minW, minW);
      atomicMax(&st0->mode, mode); atomicMin(&st0->minz, minz); atomicMax(&st0->maxz, maxz);
      atomicAdd(&st0->n_act, n_act);
      atomicMin(&st0->minx, minx); atomicMax(&st0->maxx, maxx);
      atomicMin(&st0->miny, miny); atomicMax(&st0->maxy, maxy);
    }
  }
  cl.sync();
  PNMS_CL_TRACE(1);
  const int n_act = st0->n_act, g_maxz = st0->maxz;
  const int ox = st0->minx, oy = st0->miny, g_maxx = st0->maxx, g_maxy = st0->maxy;
  const bool eligible = st0->mode == kNarrow7 && (n_act == 0 || (a.theta > 0.0 && st0->minz >= 1));
  if (!eligible) {
    cl.sync();  // every CTA has read CTA 0's statistics before any CTA exits
    if (r == 0 && threadIdx.x == 0) binned_decline(a, f);
    return;
  }
  // ---- the theta reach (pnms_binned2.cuh): a column that can suppress row i has its corner in
  // [x_i - L, x_i + z_i + 1 - R] x [y_i - L, y_i + z_i + 1 - R].  Cells taller than either
  // vertical reach (a row reaches one cell row beyond its own band) and Sy / 4 wide, cell rows
  // split into CS balanced bands
  const int g_L = n_act > 0 ? st0->maxL : 0, g_R = n_act > 0 ? st0->minW : 1;
  int Sy = max(max(g_L, g_maxz + 1 - g_R) + 1, kMinCellSide), Sx = max(Sy >> 2, kMinCellSide), GX = 1, GY = 1;
  if (n_act > 0) {
    for (;;) {
      GX = (g_maxx - ox) / Sx + 1;
      GY = (g_maxy - oy) / Sy + 1;
      if ((long long)GX * ((GY + CS - 1) / CS) + 1 <= kClCells) break;
      if (Sx < Sy) Sx *= 2;
      else { Sx *= 2; Sy *= 2; }
    }
  }
  const uint32_t Mx = div_magic(Sx), My = div_magic(Sy);
  // band o holds cell rows [rb(o), rb(o+1)), rb(o) = ceil(o*GY/CS); owner(cy) = cy*CS/GY
  auto band_lo = [&](int o) { return (o * GY + CS - 1) / CS; };
  auto owner = [&](int cy) { return (cy * CS) / GY; };
  const int my_lo = band_lo(r), my_cells = (band_lo(r + 1) - my_lo) * GX;
  // ---- pass 2: histogram on the owning CTA's counters; return value = rank in the cell
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    if (zc[k] != 0xFFFFFFFFu) {
      const int ex = (int)(xy[k] & 0xFFFFu), ey = (int)(xy[k] >> 16);
      const int cy = qdiv(ey - oy, My), cx = qdiv(ex - ox, Mx);
      const int o = owner(cy);
      const int lc = (cy - band_lo(o)) * GX + cx;
      const uint32_t rk = atomicAdd(cl.map_shared_rank(cstart, o) + lc, 1u);
      zc[k] |= ((uint32_t)lc << 16) | (min(rk, 255u) << 8);
    }
  }
  cl.sync();
  PNMS_CL_TRACE(2);
  // ---- own band: exclusive scan of the cell counts, largest cell, capacity
  {
    const int per = (my_cells + 1 + kClThreads - 1) / kClThreads;
    const int b0 = threadIdx.x * per;
    uint32_t sum = 0, big = 0;
    for (int t = 0; t < per; ++t) {
      const int c = b0 + t;
      if (c < my_cells) { sum += cstart[c]; big = max(big, cstart[c]); }
    }
    big = __reduce_max_sync(0xFFFFFFFFu, big);
    if ((threadIdx.x & 31) == 0 && big) atomicMax(&st0->big, (int)big);
    uint32_t total;
    uint32_t run = block_exclusive_scan(sum, scan_tmp, &total);
    for (int t = 0; t < per; ++t) {
      const int c = b0 + t;
      if (c < my_cells) { const uint32_t v = cstart[c]; cstart[c] = run; run += v; }
    }
    if (threadIdx.x == 0) {
      cstart[my_cells] = total;
      if (total > (uint32_t)kClCap) atomicMax(&st0->over, 1);
    }
  }
  cl.sync();
  PNMS_CL_TRACE(3);
  const bool decline = st0->big > kBinCellMax || st0->over;
  if (decline) {
    cl.sync();
  PNMS_CL_TRACE(4);
    if (r == 0 && threadIdx.x == 0) binned_decline(a, f);
    return;
  }
  // ---- pass 3: records, keys, slots and cells straight into the owner's staging arrays
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    if (zc[k] != 0xFFFFFFFFu) {
      const int el = threadIdx.x + k * kClThreads;
      const int e = e0 + el;
      const int32_t xv = (int32_t)(xy[k] & 0xFFFFu), yv = (int32_t)(xy[k] >> 16), zv = (int32_t)(zc[k] & 0xFFu);
      const int o = owner(qdiv(yv - oy, My));
      const uint32_t lc = zc[k] >> 16;
      const uint32_t pos = cl.map_shared_rank(cstart, o)[lc] + ((zc[k] >> 8) & 0xFFu);
      const RecNarrow rn = make_rec_narrow(xv, yv, zv, a.theta, kNarrow7);
      const uint64_t key = sort_key(a.s[fbase + e]);
      RecBin rb;
      rb.a = rn.a; rb.nb = rn.nb; rb.w = rn.negT | (zv + 1); rb.k = (uint32_t)(key >> 32);
      cl.map_shared_rank(tRec, o)[pos] = rb;
      cl.map_shared_rank(tKey, o)[pos] = key;
      cl.map_shared_rank(tIdx, o)[pos] = (uint16_t)e;
      cl.map_shared_rank(tCell, o)[pos] = (uint16_t)lc;
    }
  }
  cl.sync();
  PNMS_CL_TRACE(5);
  // ---- own cells in (key, slot) order: every box counts the cell members before it (no
  // serial per-cell sort on the latency path), then lands at its final position
  const int n_own = (int)cstart[my_cells];
  for (int q = threadIdx.x; q < n_own; q += kClThreads) {
    const int c = tCell[q];
    const int b = (int)cstart[c], en = (int)cstart[c + 1];
    const uint64_t kq = tKey[q];
    const uint16_t iq = tIdx[q];
    int rank = 0;
    for (int j = b; j < en; ++j) {
      const uint64_t kj = tKey[j];
      rank += kj < kq || (kj == kq && tIdx[j] < iq);
    }
    const int fpos = b + rank;
    RecBin rb = tRec[q];
    rb.w |= (en - fpos) << 8;
    recS[fpos] = rb;
    keyS[fpos] = kq;
    idxS[fpos] = iq;
  }
  cl.sync();
  PNMS_CL_TRACE(6);
  // ---- halo: the cell rows just above and below the band (the only ones a row's reach can
  // add, since S > max side) are copied once into local shared memory, next to a local copy of
  // the band, so the row scan reads shared memory only.  Extended rows [R0, R1].
  const bool pad_rule = a.d_max > cnt;
  const int my_hi = band_lo(r + 1);
  const int R0 = max(my_lo - 1, 0), R1 = min(my_hi, GY - 1);
  const int ext_rows = my_hi > my_lo ? R1 - R0 + 1 : 0;
  const int ext_cells = ext_rows * GX;
  bool ext_ok = ext_cells + 1 <= kClCells;
  int ext_n = 0, own_off = 0;
  if (ext_ok && ext_rows > 0) {
    // cell starts: every thread takes whole cells; row-major over the extended rows
    for (int c = threadIdx.x; c < ext_cells; c += kClThreads) {
      const int yy = R0 + c / GX, cx = c % GX;
      const int o = owner(yy);
      const uint32_t* cs = o == r ? cstart : cl.map_shared_rank(cstart, o);
      const int lc = (yy - band_lo(o)) * GX + cx;
      ecs[c] = cs[lc + 1] - cs[lc];  // counts first
    }
    __syncthreads();
    uint32_t total;
    {
      const int per = (ext_cells + kClThreads - 1) / kClThreads;
      const int b0 = threadIdx.x * per;
      uint32_t sum = 0;
      for (int t = 0; t < per; ++t) if (b0 + t < ext_cells) sum += ecs[b0 + t];
      uint32_t run = block_exclusive_scan(sum, scan_tmp, &total);
      for (int t = 0; t < per; ++t) {
        const int c = b0 + t;
        if (c < ext_cells) { const uint32_t v = ecs[c]; ecs[c] = run; run += v; }
      }
      if (threadIdx.x == 0) ecs[ext_cells] = total;
    }
    __syncthreads();
    ext_n = (int)total;
    own_off = (int)ecs[(my_lo - R0) * GX];
    ext_ok = ext_n <= kClCap;
    if (ext_ok) {
      // copy row by row: source range of extended row yy is contiguous in its owner's arrays
      for (int row = 0; row < ext_rows; ++row) {
        const int yy = R0 + row;
        const int o = owner(yy);
        const int lc = (yy - band_lo(o)) * GX;
        const uint32_t* cs = o == r ? cstart : cl.map_shared_rank(cstart, o);
        const int src0 = (int)cs[lc], n_row = (int)cs[lc + GX] - src0;
        const int dst0 = (int)ecs[row * GX];
        const RecBin* rr = o == r ? recS : cl.map_shared_rank(recS, o);
        const uint64_t* kr = o == r ? keyS : cl.map_shared_rank(keyS, o);
        const uint16_t* ir = o == r ? idxS : cl.map_shared_rank(idxS, o);
        for (int t = threadIdx.x; t < n_row; t += kClThreads) {
          tRec[dst0 + t] = rr[src0 + t];
          tKey[dst0 + t] = kr[src0 + t];
          tIdx[dst0 + t] = ir[src0 + t];
        }
      }
    }
    __syncthreads();
  }
  for (int p = threadIdx.x; p < n_own; p += kClThreads) {
    const RecBin ri = recS[p];
    const int32_t ix = -(int32_t)(int16_t)(ri.nb & 0xFFFFu), iy = -(int32_t)(int16_t)(ri.nb >> 16);
    const int32_t iz = (int32_t)(ri.w & 0xFF) - 1;
    const int cx0 = qdiv(max(ix - g_L - ox, 0), Mx), cy0 = qdiv(max(iy - g_L - oy, 0), My);
    const int cx1 = min(GX - 1, qdiv(ix + iz + 1 - g_R - ox, Mx)), cy1 = min(GY - 1, qdiv(iy + iz + 1 - g_R - oy, My));
    bool sup;
    if (ext_ok) {
      sup = cluster_row_scan<BY_INDEX>(ri, p + own_off, cx0, cx1, cy0, cy1, [&](int yy) { return (yy - R0) * GX; },
                                       [&](int) { return (const uint32_t*)ecs; }, [&](int) { return (const RecBin*)tRec; },
                                       [&](int) { return (const uint64_t*)tKey; },
                                       [&](int) { return (const uint16_t*)tIdx; }, [&](int) { return true; }, keyS[p],
                                       idxS[p]);
    } else {
      sup = cluster_row_scan<BY_INDEX>(
          ri, p, cx0, cx1, cy0, cy1, [&](int yy) { return (yy - band_lo(owner(yy))) * GX; },
          [&](int yy) { return (const uint32_t*)cl.map_shared_rank(cstart, owner(yy)); },
          [&](int yy) { return (const RecBin*)cl.map_shared_rank(recS, owner(yy)); },
          [&](int yy) { return (const uint64_t*)cl.map_shared_rank(keyS, owner(yy)); },
          [&](int yy) { return (const uint16_t*)cl.map_shared_rank(idxS, owner(yy)); },
          [&](int yy) { return owner(yy) == r; }, keyS[p], idxS[p]);
    }
    const int i = idxS[p];
    if (!sup && pad_rule && a.s[fbase + i] < 0.0) sup = true;
    if (!sup) {
      const int so = i / slice, il = i - so * slice;
      if (so == r) atomicOr(&kbits[il >> 5], 1u << (il & 31));
      else atomicOr(cl.map_shared_rank(kbits, so) + (il >> 5), 1u << (il & 31));
    }
  }
  cl.sync();
  PNMS_CL_TRACE(7);
  // ---- compaction (engine.py:284-293): slice popcounts -> cluster prefix -> ascending indices
  // every slice word inside the frame's W32 words is written (bits past count are zero)
  const int words_here = max(0, min(slice_words, a.W32 - e0 / 32));
  const int wpt = (words_here + kClThreads - 1) / kClThreads;
  const int w0 = threadIdx.x * wpt, w1 = min(w0 + wpt, words_here);
  uint32_t local = 0;
  for (int w = w0; w < w1; ++w) {
    const uint32_t bits = kbits[w];
    local += __popc(bits);
    if (a.keep_mask) a.keep_mask[(long long)f * a.W32 + e0 / 32 + w] = bits;
  }
  uint32_t total;
  uint32_t pos = block_exclusive_scan(local, scan_tmp, &total);
  if (threadIdx.x == 0) st0->total[r] = total;
  cl.sync();
  PNMS_CL_TRACE(8);
  uint32_t base = 0;
  for (int o = 0; o < r; ++o) base += st0->total[o];
  if (a.keep_idx) {
    for (int w = w0; w < w1; ++w) {
      uint32_t bits = kbits[w];
      while (bits) {
        a.keep_idx[fbase + base + pos++] = e0 + w * 32 + __ffs(bits) - 1;
        bits &= bits - 1;
      }
    }
  }
  if (r == CS - 1 && threadIdx.x == 0) {
    if (a.keep_count) a.keep_count[f] = (int32_t)(base + total);
    a.fallback[f] = 0;
  }
  cl.sync();  // CTA 0's statistics are read until here
  PNMS_CL_TRACE(9);
}

}  // namespace pnms

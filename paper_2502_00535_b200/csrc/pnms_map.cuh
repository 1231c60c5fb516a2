// pnms_map.cuh — the pairwise overlap map (engine.py:204-244), restricted to gate-passing
// pairs by the score sort, fused with the row reduction (engine.py:253-281).
//
// Reference: fill_rows() evaluates every ordered cell (i, j) of the d_max x d_max matrix,
// stores keep|~gate bits, and reduce_phase() ANDs each row.  Here sorted row p only visits
// columns q < lim[p] (the cells whose gate passes) and keeps, per row, the OR of
// "j suppresses i" in registers; the bit matrix is never materialised.  Per row the warp
// ballot of the final verdicts is OR-ed into a 32-bit word of the frame's suppression mask.
//
// Work decomposition: a work item is (frame, row block of kMapWarps*32*R sorted rows, column
// chunk of `chunk` columns).  The CTA stages its column chunk into shared memory with one
// bulk async copy (cp.async.bulk, TMA engine) and each warp scans it for 32*R rows (R rows
// per lane, the column record broadcast from shared memory).  Columns are visited in
// descending position (nearest scores first) so suppressed rows end early; a warp stops as
// soon as all its rows are decided.  Items are ordered heaviest-first within a frame.
//
// Narrow8 inner step (per row, per column) — 3 ALU-pipe + 2 FMA-pipe instructions:
//   t1 = VIADDMNMX.S16x2      min(a_i + nb_j, zz_i)          = min(xe1_i - x_j, z_i+1)
//   t2 = VIADDMNMX.S16x2.RELU max(min(a_j + nb_i, t1), 0)    = .. min(xe1_j - x_i)
//   v  = VIMNMX.S16x2.RELU    min(t2, zz_j)                  -> (w, h) packed, exact
//   s  = IMAD                 v * 65536                      = w << 16
//   d  = IMAD.HI.U32          hi32(v*s + {zz_j, negT_j})     = w*h - T_j   (w <= 255)
//   acc &= d   (LOP3, 3-input: one per two columns)          sign clear <=> suppressed
#pragma once
#include "pnms_common.cuh"

namespace pnms {

struct MapArgs {
  const uint8_t* rec;
  const int32_t* lim;
  uint32_t* supp;
  const FrameMeta* meta;
  int batch, n_max, W32;
  int rows_per_block;   // kMapWarps * 32 * R
  int chunk;            // columns per work item
  int n_rb;             // row blocks per frame
  int items_per_frame;
  uint32_t k65536;      // 65536, passed at run time so the multiply stays on the FMA pipe
};

// number of column chunks of row block rb: its rows' limits are < (rb+1)*RB
__device__ __forceinline__ int chunks_of(int rb, int RB, int chunk, int n_max) {
  int cols = min((rb + 1) * RB - 1, n_max);
  return (cols + chunk - 1) / chunk;
}

template <int R>
struct RowState {
  uint32_t a[R], nb[R], zz[R];
  int acc[R];       // narrow: AND of (w*h - T); sign bit clear once a suppressor was seen
  int lim[R];
  bool active[R];
  bool pre[R];      // already suppressed by another work item
};

template <int R>
__device__ __forceinline__ bool rows_done_narrow(const RowState<R>& st) {
  bool done = true;
#pragma unroll
  for (int r = 0; r < R; ++r) done &= (!st.active[r]) | st.pre[r] | (st.acc[r] >= 0);
  return done;
}

// --- narrow (s16x2) column scans -------------------------------------------------------
template <int R, bool kNarrow8>
__device__ __forceinline__ void pair_narrow(RowState<R>& st, const uint4 c, uint32_t k65536) {
#pragma unroll
  for (int r = 0; r < R; ++r) {
    uint32_t t1 = __viaddmin_s16x2(st.a[r], c.y, st.zz[r]);
    uint32_t t2 = __viaddmin_s16x2_relu(c.x, st.nb[r], t1);
    uint32_t v = __vimin_s16x2_relu(t2, c.z);
    int d;
    if (kNarrow8) {
      uint32_t s = v * k65536;
      const uint64_t addend = ((uint64_t)c.w << 32) | c.z;
      d = (int)(uint32_t)(((uint64_t)v * s + addend) >> 32);
    } else {
      d = (int)((v & 0xFFFFu) * (v >> 16)) + (int)c.w;
    }
    st.acc[r] &= d;
  }
}

template <int R, bool kNarrow8>
__device__ __forceinline__ void pair_narrow_masked(RowState<R>& st, const uint4 c, int q, uint32_t k65536) {
#pragma unroll
  for (int r = 0; r < R; ++r) {
    uint32_t t1 = __viaddmin_s16x2(st.a[r], c.y, st.zz[r]);
    uint32_t t2 = __viaddmin_s16x2_relu(c.x, st.nb[r], t1);
    uint32_t v = __vimin_s16x2_relu(t2, c.z);
    int d;
    if (kNarrow8) {
      uint32_t s = v * k65536;
      const uint64_t addend = ((uint64_t)c.w << 32) | c.z;
      d = (int)(uint32_t)(((uint64_t)v * s + addend) >> 32);
    } else {
      d = (int)((v & 0xFFFFu) * (v >> 16)) + (int)c.w;
    }
    st.acc[r] &= (q < st.lim[r]) ? d : -1;
  }
}

template <int R, bool kNarrow8>
__device__ __forceinline__ void scan_narrow(RowState<R>& st, const uint4* scol, int c0, int m_lo, int m_hi,
                                            int u_hi, uint32_t k65536) {
  // masked tail: columns [m_lo, m_hi) where some rows of the warp are past their limit
  for (int q = m_hi - 1; q >= m_lo; --q) pair_narrow_masked<R, kNarrow8>(st, scol[q - c0], q, k65536);
  if (__all_sync(0xFFFFFFFFu, rows_done_narrow(st))) return;
  // unmasked body: columns [c0, u_hi), descending, decided-check every 32 columns
  for (int qb = u_hi; qb > c0; qb -= 32) {
    const int qlo = max(c0, qb - 32);
    int q = qb - 1;
    for (; q - 7 >= qlo; q -= 8) {
      uint4 cc[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) cc[u] = scol[q - u - c0];
#pragma unroll
      for (int u = 0; u < 8; ++u) pair_narrow<R, kNarrow8>(st, cc[u], k65536);
    }
    for (; q >= qlo; --q) pair_narrow<R, kNarrow8>(st, scol[q - c0], k65536);
    if (__all_sync(0xFFFFFFFFu, rows_done_narrow(st))) return;
  }
}

// --- wide (exact int32-wrap / float64 emulation) -----------------------------------------
__device__ __forceinline__ bool suppress_wide(const RecWide& ri, const RecWide& cj) {
  int32_t wv = (int32_t)((uint32_t)min(ri.xe, cj.xe) - (uint32_t)max(ri.x, cj.x) + 1u);
  int32_t hv = (int32_t)((uint32_t)min(ri.ye, cj.ye) - (uint32_t)max(ri.y, cj.y) + 1u);
  wv = max(wv, 0);
  hv = max(hv, 0);
  double prod = __dmul_rn((double)wv, (double)hv);
  return !(prod < cj.thr);
}

template <int R>
__device__ __noinline__ void warp_scan_wide(const MapArgs& a, const RecWide* scol, const RecWide* rec_frame, int c0,
                                            int c1, int pw, int p_end, const int32_t* lim_frame,
                                            bool (&hit)[R], const bool (&pre)[R]) {
  const int lane = threadIdx.x & 31;
  RecWide ri[R];
  int lim[R];
  bool active[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int p = pw + r * 32 + lane;
    active[r] = p < p_end;
    lim[r] = active[r] ? lim_frame[p] : 0;
    if (active[r]) ri[r] = rec_frame[p];
    hit[r] = false;
  }
  for (int q = c1 - 1; q >= c0; --q) {
    const RecWide cj = scol[q - c0];
#pragma unroll
    for (int r = 0; r < R; ++r)
      if (active[r] && !hit[r] && !pre[r] && q < lim[r]) hit[r] = suppress_wide(ri[r], cj);
    if (((q - c0) & 31) == 0) {
      bool done = true;
#pragma unroll
      for (int r = 0; r < R; ++r) done &= (!active[r]) | hit[r] | pre[r];
      if (__all_sync(0xFFFFFFFFu, done)) break;
    }
  }
}

template <int R>
__global__ void __launch_bounds__(kMapWarps * 32) pnms_map_kernel(MapArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bar;
  const int f = blockIdx.x / a.items_per_frame;
  int item = blockIdx.x % a.items_per_frame;
  const int RB = a.rows_per_block;
  int rb = a.n_rb - 1;
  for (; rb > 0; --rb) {
    const int nc = chunks_of(rb, RB, a.chunk, a.n_max);
    if (item < nc) break;
    item -= nc;
  }
  const int c = item;
  const FrameMeta fm = a.meta[f];
  const int n_act = fm.n_active;
  const int p_lo = rb * RB;
  if (p_lo >= n_act) return;
  const int p_end = min(p_lo + RB, n_act);
  const long long fbase = (long long)f * a.n_max;
  const int32_t* lim_frame = a.lim + fbase;
  const int c0 = c * a.chunk;
  const int c1 = min(c0 + a.chunk, lim_frame[p_end - 1]);
  if (c0 >= c1) return;

  const int mode = fm.mode;
  const int rec_sz = (mode == kWide) ? (int)sizeof(RecWide) : (int)sizeof(RecNarrow);
  const uint8_t* rec_frame = a.rec + fbase * kRecBytes;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    const uint32_t bytes = (uint32_t)(c1 - c0) * rec_sz;
    mbar_expect_tx(&bar, bytes);
    bulk_g2s(smem_raw, rec_frame + (size_t)c0 * rec_sz, bytes, &bar);
  }
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int pw = p_lo + warp * 32 * R;
  mbar_wait(&bar, 0);
  if (pw >= p_end) return;
  const int p_last = min(pw + 32 * R, p_end) - 1;
  const int lim_lo = lim_frame[pw], lim_hi = lim_frame[p_last];
  uint32_t* supp_frame = a.supp + (long long)f * a.W32;

  bool pre[R];
  bool all_pre = true;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int p = pw + r * 32 + lane;
    const int wi = (pw >> 5) + r;
    uint32_t wbits = (wi < a.W32) ? *((volatile uint32_t*)(supp_frame + wi)) : 0u;
    pre[r] = (p < p_end) && ((wbits >> lane) & 1u);
    all_pre &= (p >= p_end) | pre[r];
  }
  if (__all_sync(0xFFFFFFFFu, all_pre)) return;

  bool sup[R];
  if (mode == kWide) {
    bool hit[R];
    warp_scan_wide<R>(a, reinterpret_cast<const RecWide*>(smem_raw), reinterpret_cast<const RecWide*>(rec_frame),
                      c0, min(c1, lim_hi), pw, p_end, lim_frame, hit, pre);
#pragma unroll
    for (int r = 0; r < R; ++r) sup[r] = hit[r];
  } else {
    RowState<R> st;
    const RecNarrow* rf = reinterpret_cast<const RecNarrow*>(rec_frame);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int p = pw + r * 32 + lane;
      st.active[r] = p < p_end;
      st.pre[r] = pre[r];
      RecNarrow rr = st.active[r] ? rf[p] : RecNarrow{0u, 0u, 0u, 0};
      st.a[r] = rr.a;
      st.nb[r] = rr.nb;
      st.zz[r] = rr.zz;
      st.lim[r] = st.active[r] ? lim_frame[p] : 0;
      st.acc[r] = -1;
    }
    const uint4* scol = reinterpret_cast<const uint4*>(smem_raw);
    const int m_lo = max(c0, lim_lo), m_hi = min(c1, lim_hi);
    const int u_hi = min(c1, lim_lo);
    if (mode == kNarrow8)
      scan_narrow<R, true>(st, scol, c0, m_lo, m_hi, u_hi, a.k65536);
    else
      scan_narrow<R, false>(st, scol, c0, m_lo, m_hi, u_hi, a.k65536);
#pragma unroll
    for (int r = 0; r < R; ++r) sup[r] = st.active[r] && st.acc[r] >= 0;
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const uint32_t bits = __ballot_sync(0xFFFFFFFFu, sup[r] && !pre[r]);
    if (lane == 0 && bits) atomicOr(supp_frame + (pw >> 5) + r, bits);
  }
}

}  // namespace pnms

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
// bulk async copy (cp.async.bulk, TMA engine) and each warp scans it for 32*R rows: lane l
// owns rows p0 + 32*g + l for the R row groups g.  Columns are visited in descending position
// (nearest scores first).  Because lim[] is monotone in p, the column range splits into
// per-group segments: in [lim_lo[g], lim_hi[g]) only group g needs a per-row mask, groups
// above g are fully active and groups below are idle — no work is spent on masked-off pairs
// beyond one 32-column band per group.  A warp stops once every row is decided.
//
// Narrow7 inner step (per row, per column; sides <= 126, coordinates < 32768):
//   t1 = VIADDMNMX.S16x2       min(a_i + nb_j, zz_i)          = min(xe1_i - x_j, z_i+1)
//   t2 = VIADDMNMX.S16x2.RELU  max(min(a_j + nb_i, t1), 0)    .. min(xe1_j - x_i)
//   v  = VIMNMX.S16x2.RELU     min(t2, zz_j)                  -> (w, h) packed, exact
//   d  = IMAD                  v*v - T_j*2^17                 = w^2 + (w*h - T_j)*2^17
//   acc &= d   (LOP3, 3-input: one per two columns)           sign clear <=> suppressed
// v*v mod 2^32 = w^2 + w*h*2^17 because h^2*2^32 vanishes; with w, h <= 127 nothing
// overflows and w^2 < 2^17, so sign(d) = sign(w*h - T_j) with w*h == T_j giving d >= 0.
// That is 3 ALU-pipe SIMD ops + 1 full-rate FMA-pipe IMAD + 1/2 LOP3 per pair.
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
  const uint8_t* dense;   // optional [batch]: process frame f only if dense[f] != 0
  const int32_t* list;    // optional: process only frames list[0 .. *list_count) (grid-stride)
  const int* list_count;
};

// number of column chunks of row block rb: its rows' limits are < (rb+1)*RB
__device__ __forceinline__ int chunks_of(int rb, int RB, int chunk, int n_max) {
  int cols = min((rb + 1) * RB - 1, n_max);
  return (cols + chunk - 1) / chunk;
}

template <int R>
struct NarrowRows {
  uint32_t a[R], nb[R], zz[R];
  int acc[R];   // AND of d over the visited columns; >= 0 once decided (suppressed)
  int lim[R];
};

template <int R>
__device__ __forceinline__ bool all_decided(const NarrowRows<R>& st) {
  bool done = true;
#pragma unroll
  for (int r = 0; r < R; ++r) done &= st.acc[r] >= 0;
  return __all_sync(0xFFFFFFFFu, done);
}

template <int MODE>
__device__ __forceinline__ int pair_d(uint32_t a_i, uint32_t nb_i, uint32_t zz_i, const uint4& c) {
  const uint32_t t1 = __viaddmin_s16x2(a_i, c.y, zz_i);
  const uint32_t t2 = __viaddmin_s16x2_relu(c.x, nb_i, t1);
  const uint32_t v = __vimin_s16x2_relu(t2, c.z);
  if (MODE == kNarrow7) return (int)(v * v) + (int)c.w;
  return (int)((v & 0xFFFFu) * (v >> 16)) + (int)c.w;
}

// Columns [q_lo, q_hi), descending.  Row groups [G, R) take part; with MASK the rows of group
// G only count columns below their own limit.  Returns true once every row is decided.
template <int R, int MODE, int G, bool MASK>
__device__ __forceinline__ bool scan_segment(NarrowRows<R>& st, const uint4* scol, int c0, int q_lo, int q_hi) {
  int q = q_hi - 1;
  while (q >= q_lo) {
    const int stop = max(q_lo, q - 63);
    for (; q - 7 >= stop; q -= 8) {
      uint4 cc[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) cc[u] = scol[q - u - c0];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
#pragma unroll
        for (int r = G; r < R; ++r) {
          const int d = pair_d<MODE>(st.a[r], st.nb[r], st.zz[r], cc[u]);
          if (MASK && r == G) st.acc[r] &= (q - u < st.lim[r]) ? d : -1;
          else st.acc[r] &= d;
        }
      }
    }
    for (; q >= stop; --q) {
      const uint4 c = scol[q - c0];
#pragma unroll
      for (int r = G; r < R; ++r) {
        const int d = pair_d<MODE>(st.a[r], st.nb[r], st.zz[r], c);
        if (MASK && r == G) st.acc[r] &= (q < st.lim[r]) ? d : -1;
        else st.acc[r] &= d;
      }
    }
    if (all_decided(st)) return true;
  }
  return false;
}

// Walk the per-group segments from the highest row group down (see header comment).
template <int R, int MODE, int G>
__device__ __forceinline__ bool scan_groups(NarrowRows<R>& st, const uint4* scol, int c0, int c1,
                                            const int (&lim_lo)[R], const int (&lim_hi)[R]) {
  if (scan_segment<R, MODE, G, true>(st, scol, c0, max(c0, lim_lo[G]), min(c1, lim_hi[G]))) return true;
  const int below = (G > 0) ? lim_hi[G > 0 ? G - 1 : 0] : c0;
  if (scan_segment<R, MODE, G, false>(st, scol, c0, max(c0, below), min(c1, lim_lo[G]))) return true;
  if constexpr (G > 0) return scan_groups<R, MODE, G - 1>(st, scol, c0, c1, lim_lo, lim_hi);
  return false;
}

template <int R, int MODE>
__device__ __forceinline__ void warp_scan_narrow(const RecNarrow* rf, const uint4* scol, const int32_t* lim_frame,
                                                 int c0, int c1, int pw, int p_end, const bool (&pre)[R],
                                                 bool (&sup)[R]) {
  const int lane = threadIdx.x & 31;
  NarrowRows<R> st;
  int lim_lo[R], lim_hi[R];
  int last_hi = 0;
#pragma unroll
  for (int g = 0; g < R; ++g) {
    const int p = pw + g * 32 + lane;
    const bool active = p < p_end;
    const RecNarrow rr = active ? rf[p] : RecNarrow{0u, 0u, 0u, 0};
    st.a[g] = rr.a;
    st.nb[g] = rr.nb;
    st.zz[g] = rr.zz;
    st.lim[g] = active ? lim_frame[p] : 0;
    st.acc[g] = (!active || pre[g]) ? 0 : -1;
    const int g0 = pw + g * 32;
    if (g0 < p_end) {
      lim_lo[g] = lim_frame[g0];
      lim_hi[g] = lim_frame[min(g0 + 31, p_end - 1)];
      last_hi = lim_hi[g];
    } else {
      lim_lo[g] = lim_hi[g] = last_hi;  // idle group: empty segments
    }
  }
  scan_groups<R, MODE, R - 1>(st, scol, c0, c1, lim_lo, lim_hi);
#pragma unroll
  for (int g = 0; g < R; ++g) sup[g] = (pw + g * 32 + lane < p_end) && !pre[g] && st.acc[g] >= 0;
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
static __device__ __noinline__ void warp_scan_wide(const RecWide* scol, const RecWide* rec_frame, int c0, int c1, int pw,
                                            int p_end, const int32_t* lim_frame, bool (&hit)[R],
                                            const bool (&pre)[R]) {
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
__device__ __forceinline__ void map_item(const MapArgs& a, int f, int item, unsigned char* smem_raw, uint64_t& bar) {
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
    warp_scan_wide<R>(reinterpret_cast<const RecWide*>(smem_raw), reinterpret_cast<const RecWide*>(rec_frame), c0,
                      min(c1, lim_frame[p_last]), pw, p_end, lim_frame, sup, pre);
  } else {
    const RecNarrow* rf = reinterpret_cast<const RecNarrow*>(rec_frame);
    const uint4* scol = reinterpret_cast<const uint4*>(smem_raw);
    if (mode == kNarrow7)
      warp_scan_narrow<R, kNarrow7>(rf, scol, lim_frame, c0, c1, pw, p_end, pre, sup);
    else
      warp_scan_narrow<R, kNarrow16>(rf, scol, lim_frame, c0, c1, pw, p_end, pre, sup);
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const uint32_t bits = __ballot_sync(0xFFFFFFFFu, sup[r] && !pre[r]);
    if (lane == 0 && bits) atomicOr(supp_frame + (pw >> 5) + r, bits);
  }
}

template <int R>
__global__ void __launch_bounds__(kMapWarps * 32) pnms_map_kernel(MapArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bar;
  const int f = blockIdx.x / a.items_per_frame;
  if (a.dense && !a.dense[f]) return;
  map_item<R>(a, f, blockIdx.x % a.items_per_frame, smem_raw, bar);
}

// the same over the binned path's declined-frame list (persistent grid, programmatic
// dependent launch); a separate kernel so the full-batch one keeps its register budget
template <int R>
__global__ void __launch_bounds__(kMapWarps * 32) pnms_map_kernel_list(MapArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ __align__(8) uint64_t bar;
  pdl_wait();  // PDL: the previous kernel's results are visible after this
  pdl_trigger();
  const long long n = (long long)*a.list_count * a.items_per_frame;
  for (long long it = blockIdx.x; it < n; it += gridDim.x) {
    map_item<R>(a, a.list[it / a.items_per_frame], (int)(it % a.items_per_frame), smem_raw, bar);
    __syncthreads();  // every warp is past the barrier wait and done with the column chunk
  }
}

}  // namespace pnms

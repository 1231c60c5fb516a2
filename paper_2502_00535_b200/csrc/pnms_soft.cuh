// pnms_soft.cuh — Soft-NMS rescoring (oracles.soft_nms_rescore, oracles.py:88-123) on the
// device, bit-identical to the reference's sequential loop in both modes.
//
// Reference semantics: repeatedly select the pending detection with the highest current
// score (ties: lowest index), remove it from the pending set, and multiply every pending
// score by a factor of its coverage by the selected box, cov = w*h / (z_sel+1)^2
// (oracles.py:31-34, clamped inclusive extents, a correctly rounded float64 quotient):
//   linear:   s *= 1 - cov   when cov >= theta
//   gaussian: s *= exp(-(cov*cov) / sigma)
// Non-overlapping pairs have cov = 0 and factor exactly 1.0, so only overlapping pairs
// interact.
//
// Parallel exact resolution.  Factors are <= 1 and scores positive, so scores only fall and
// the selection keys (-score at selection, index) strictly increase along the reference's
// sequence.  Hence a box's final score is its initial score times the factors of the
// overlapping boxes selected before it, applied in selection order.  Every round, each
// pending box recomputes its tentative score from its already-final overlapping neighbours
// in key order (an upper bound of its final score, exact once nothing pending can precede
// it), and a pending box whose (tentative score, index) key precedes the keys of all its
// pending overlapping neighbours is final: nothing pending can be selected before it.  The
// box with the globally smallest key always qualifies, so every round finalizes at least one
// box; typical frames finish in a handful of rounds.  After kSoftMaxRounds rounds (dense
// crowds) the remaining boxes are finished by the reference's own one-at-a-time loop.
//
// Candidates come from spatial cells of side max_z + 1 (3x3 neighbourhood, exact because
// zero overlap never changes a score); frames with negative coordinates or a crowded cell
// use every slot.  Scores must be finite and > 0 (the validated domain, detections.py:79-84);
// frames outside it are flagged in `status` and left unwritten.  Gaussian mode evaluates
// exp with glibc_exp (pnms_libm.cuh), a restatement of the host libm exp the reference's
// math.exp calls, so its scores are bit-identical too.
#pragma once
#include "pnms_libm.cuh"
#include "pnms_common.cuh"

namespace pnms {

constexpr int kSoftThreads = 512;
constexpr int kSoftMaxSlots = 4096;     // largest frame whose state fits shared memory
constexpr int kSoftMaxCells = 65535;    // cell ids are 16-bit
constexpr int kSoftCellMax = 64;
constexpr int kSoftMaxRounds = 96;

enum SoftState : uint8_t { kSoftPending = 0, kSoftReady = 1, kSoftFinal = 2 };

struct SoftArgs {
  const int32_t *x, *y, *z;
  const double* s;
  const int32_t* counts;
  int batch, n_max;
  int mode;        // 0 linear, 1 gaussian
  double theta, sigma;
  double* out_s;   // [batch, n_max] rescored scores (0.0 in padding slots)
  int32_t* status; // [batch] 0 ok, 1 scores outside the domain (frame left unwritten)
  int32_t* rounds; // optional [batch] rounds used (diagnostics)
  unsigned char* scratch;  // GLOBAL: [batch] slices of scratch_stride bytes (soft_smem_bytes)
  size_t scratch_stride;
};

__host__ __device__ inline int soft_npad(int n_max) { return (n_max + 127) & ~127; }
inline size_t soft_smem_bytes(int n_max) {
  const size_t n = (size_t)soft_npad(n_max);
  const size_t cells = n < 32 ? 64 : 2 * n;  // rectangular cells: up to two per box
  return (n * (4 * 3 + 8 + 8 + 8 + 1 + 1 + 2 + 2 + 2 + 2 + 2) + (cells + 4) * 4 + 64 * 4 + 64 + 255) / 256 * 256;
}
__host__ __device__ inline int soft_max_cells(int npad) {
  const int c = npad < 32 ? 64 : 2 * npad;
  return c > kSoftMaxCells ? kSoftMaxCells : c;
}

// the reference's factor of box b on pending box j (oracles.py:31-34, 115-120); `ovl` is
// false when the boxes do not overlap (factor exactly 1.0)
__device__ __forceinline__ double soft_apply(bool small, double sj, int32_t jx, int32_t jy, int32_t jz, int32_t bx,
                                             int32_t by, int32_t bz, int mode, double theta, double sigma) {
  if (small) {
    const int w = min(jx + jz, bx + bz) - max(jx, bx) + 1;
    const int h = min(jy + jz, by + bz) - max(jy, by) + 1;
    if (w <= 0 || h <= 0) return sj;
    const double cov = __ddiv_rn(__int2double_rn(w * h), __int2double_rn((bz + 1) * (bz + 1)));
    if (mode == 0) return cov >= theta ? __dmul_rn(sj, __dsub_rn(1.0, cov)) : sj;
    return __dmul_rn(sj, glibc_exp(__ddiv_rn(-__dmul_rn(cov, cov), sigma)));
  }
  const long long w = min((long long)jx + jz, (long long)bx + bz) - (long long)max(jx, bx) + 1;
  const long long h = min((long long)jy + jz, (long long)by + bz) - (long long)max(jy, by) + 1;
  if (w <= 0 || h <= 0) return sj;
  const long long area = ((long long)bz + 1) * ((long long)bz + 1);
  const double cov = __ddiv_rn(__ll2double_rn(w * h), __ll2double_rn(area));
  if (mode == 0) return cov >= theta ? __dmul_rn(sj, __dsub_rn(1.0, cov)) : sj;
  return __dmul_rn(sj, glibc_exp(__ddiv_rn(-__dmul_rn(cov, cov), sigma)));  // math.exp, bit for bit
}

// `small`: every coordinate and side of the frame is >= 0 and x + z, y + z < 2^15, so the
// extents and the area product are exact in 32 bits (the 64-bit forms serve every other frame)
__device__ __forceinline__ bool soft_overlap(bool small, int32_t ax, int32_t ay, int32_t az, int32_t bx, int32_t by,
                                             int32_t bz) {
  if (small) {
    const int w = min(ax + az, bx + bz) - max(ax, bx) + 1;
    const int h = min(ay + az, by + bz) - max(ay, by) + 1;
    return (w > 0) & (h > 0);
  }
  const long long w = min((long long)ax + az, (long long)bx + bz) - (long long)max(ax, bx) + 1;
  const long long h = min((long long)ay + az, (long long)by + bz) - (long long)max(ay, by) + 1;
  return w > 0 && h > 0;
}

// (key, index) order: the reference's selection order (oracles.py:113, min over (-s, i))
__device__ __forceinline__ bool soft_before(uint64_t ka, int ia, uint64_t kb, int ib) {
  return ka < kb || (ka == kb && ia < ib);
}

struct SoftFrame {
  int32_t *sx, *sy, *sz;
  double *s0, *cur;
  uint64_t* fkey;          // sort_key(cur) of every box (the selection key once final)
  uint8_t *state, *mark;   // mark: ready this round (written only by the box's own thread)
  uint16_t *cellof, *list;
  uint16_t* fround;         // round in which the box became final
  uint32_t* cstart;   // after the scatter: cstart[c] = end(c) = start(c+1), start(0) = 0
  int cnt, GX, GY, Sx, Sy, ox, oy, maxz;
  bool bin, small;

  // visit every candidate slot that may overlap box j: the cells its overlapping boxes'
  // corners can lie in ([x - max_z, x + z] x [y - max_z, y + z]; cells Sx wide and Sy tall,
  // one contiguous run per cell row), or every slot
  template <class F>
  __device__ __forceinline__ void for_candidates(int j, F&& fn) const {
    if (bin) {
      int cx0, cy0, cx1, cy1;
      if (small) {  // 32-bit quotients (the 64-bit division is a long software sequence)
        const int jx = sx[j], jy = sy[j], jz = sz[j];
        cx0 = (int)((uint32_t)max(0, jx - maxz - ox) / (uint32_t)Sx);
        cy0 = (int)((uint32_t)max(0, jy - maxz - oy) / (uint32_t)Sy);
        cx1 = min(GX - 1, (int)((uint32_t)(jx + jz - ox) / (uint32_t)Sx));
        cy1 = min(GY - 1, (int)((uint32_t)(jy + jz - oy) / (uint32_t)Sy));
      } else {
        const long long jx = sx[j], jy = sy[j], jz = sz[j];
        cx0 = (int)(max(0LL, jx - maxz - ox) / Sx);
        cy0 = (int)(max(0LL, jy - maxz - oy) / Sy);
        cx1 = (int)min((long long)GX - 1, (jx + jz - ox) / Sx);
        cy1 = (int)min((long long)GY - 1, (jy + jz - oy) / Sy);
      }
      for (int yy = cy0; yy <= cy1; ++yy) {
        const int c0 = yy * GX + cx0, c1 = yy * GX + cx1;
        const int b = c0 == 0 ? 0 : (int)cstart[c0 - 1], en = (int)cstart[c1];
        for (int q = b; q < en; ++q) fn((int)list[q]);
      }
    } else {
      for (int q = 0; q < cnt; ++q) fn(q);
    }
  }
};

// GLOBAL: the per-slot state lives in a global workspace slice instead of shared memory
// (frames above kSoftMaxSlots; same layout, same code)
template <bool GLOBAL>
__global__ void __launch_bounds__(kSoftThreads) pnms_soft_frame(SoftArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int s_stat[10];  // 0 minx 1 miny 2 maxx 3 maxy 4 maxz 5 bin_ok 6 big 7 pending 8 bad 9 arg
  __shared__ unsigned long long s_best[kSoftThreads / 32];
  __shared__ uint32_t scan_tmp[64];
  const int f = blockIdx.x;
  const long long fbase = (long long)f * a.n_max;
  const int cnt = frame_count(a.counts, f, a.n_max);
  const int npad = soft_npad(a.n_max);
  const int max_cells = soft_max_cells(npad);
  unsigned char* base;
  if constexpr (GLOBAL) base = a.scratch + (size_t)f * a.scratch_stride;
  else base = smem_raw;
  SoftFrame F;
  F.sx = reinterpret_cast<int32_t*>(base);
  F.sy = F.sx + npad;
  F.sz = F.sy + npad;
  F.s0 = reinterpret_cast<double*>(F.sz + npad);
  F.cur = F.s0 + npad;
  F.fkey = reinterpret_cast<uint64_t*>(F.cur + npad);
  F.state = reinterpret_cast<uint8_t*>(F.fkey + npad);
  F.mark = F.state + npad;
  F.cellof = reinterpret_cast<uint16_t*>(F.mark + npad);
  F.list = F.cellof + npad;
  F.fround = F.list + npad;
  uint16_t* plist[2] = {F.fround + npad, F.fround + 2 * npad};  // pending boxes, double-buffered
  F.cstart = reinterpret_cast<uint32_t*>(F.fround + 3 * npad);
  F.cnt = cnt;

  if (threadIdx.x == 0) {
    s_stat[0] = s_stat[1] = 0x7FFFFFFF;
    s_stat[2] = s_stat[3] = -0x7FFFFFFF;
    s_stat[4] = 0; s_stat[5] = 1; s_stat[6] = 0; s_stat[7] = 0; s_stat[8] = 0;
  }
  __syncthreads();
  // ---- load
  for (int e = threadIdx.x; e < cnt; e += kSoftThreads) {
    const long long g = fbase + e;
    const int32_t xv = a.x[g], yv = a.y[g], zv = a.z[g];
    const double sv = a.s[g];
    F.sx[e] = xv; F.sy[e] = yv; F.sz[e] = zv;
    F.s0[e] = sv; F.cur[e] = sv; F.fkey[e] = sort_key(sv);
    F.state[e] = kSoftPending; F.mark[e] = 0; F.fround[e] = 0xFFFF;
    if (!(sv > 0.0 && sv <= 1.7976931348623157e308)) atomicOr(&s_stat[8], 1);
    if (xv < 0 || yv < 0 || zv < 0) atomicAnd(&s_stat[5], 0);
    atomicMin(&s_stat[0], xv); atomicMin(&s_stat[1], yv);
    atomicMax(&s_stat[2], xv); atomicMax(&s_stat[3], yv); atomicMax(&s_stat[4], zv);
  }
  __syncthreads();
  if (s_stat[8]) {
    if (threadIdx.x == 0) a.status[f] = 1;
    return;
  }
  // ---- spatial cells (exact: zero overlap leaves a score unchanged)
  F.bin = s_stat[5] != 0 && cnt > 0;
  F.Sx = F.Sy = 1; F.GX = 1; F.GY = 1;
  F.ox = s_stat[0]; F.oy = s_stat[1]; F.maxz = s_stat[4];
  F.small = s_stat[5] != 0 && (long long)s_stat[2] + s_stat[4] < 32768 && (long long)s_stat[3] + s_stat[4] < 32768;
  if (F.bin) {  // cells Sx wide, Sy tall, as pnms_greedy.cuh
    F.Sy = s_stat[4] + 1;
    if (F.Sy <= 0) F.bin = false;
    F.Sx = max(F.Sy >> 2, 1);
  }
  if (F.bin) {
    for (;;) {
      F.GX = (int)(((long long)s_stat[2] - F.ox) / F.Sx + 1);
      F.GY = (int)(((long long)s_stat[3] - F.oy) / F.Sy + 1);
      if ((long long)F.GX * F.GY <= max_cells) break;
      if (F.Sy > (1 << 29)) { F.GX = F.GY = 1; break; }
      if (F.Sx < F.Sy) F.Sx *= 2;
      else { F.Sx *= 2; F.Sy *= 2; }
    }
    const int cells = F.GX * F.GY;
    for (int c = threadIdx.x; c <= cells; c += kSoftThreads) F.cstart[c] = 0u;
    __syncthreads();
    for (int e = threadIdx.x; e < cnt; e += kSoftThreads) {
      // (binned frames have non-negative coordinates: the offsets and quotients fit 32 bits)
      const int c = (int)((uint32_t)(F.sy[e] - F.oy) / (uint32_t)F.Sy) * F.GX +
                    (int)((uint32_t)(F.sx[e] - F.ox) / (uint32_t)F.Sx);
      F.cellof[e] = (uint16_t)c;
      atomicAdd(&F.cstart[c], 1u);
    }
    __syncthreads();
    {
      const int per = (cells + 1 + kSoftThreads - 1) / kSoftThreads;
      const int b0 = threadIdx.x * per;
      uint32_t sum = 0, big = 0;
      for (int t = 0; t < per; ++t) {
        const int c = b0 + t;
        if (c < cells) { sum += F.cstart[c]; big = max(big, F.cstart[c]); }
      }
      big = __reduce_max_sync(0xFFFFFFFFu, big);
      if ((threadIdx.x & 31) == 0) atomicMax(&s_stat[6], (int)big);
      uint32_t run = block_exclusive_scan(sum, scan_tmp, nullptr);
      for (int t = 0; t < per; ++t) {
        const int c = b0 + t;
        if (c < cells) { const uint32_t v = F.cstart[c]; F.cstart[c] = run; run += v; }
      }
    }
    __syncthreads();
    F.bin = s_stat[6] <= kSoftCellMax;
    if (F.bin) {
      for (int e = threadIdx.x; e < cnt; e += kSoftThreads) {
        const uint32_t pos = atomicAdd(&F.cstart[F.cellof[e]], 1u);
        F.list[pos] = (uint16_t)e;
      }
    }
  }
  __syncthreads();

  const int mode = a.mode;
  const double theta = a.theta, sigma = a.sigma;
  // ---- rounds over a compacted list of the pending boxes.  Every phase writes only the slots
  // of its own boxes and reads the others' slots as the previous barrier left them
  // (race-free by construction).
  __shared__ int s_npend[2];
  for (int e = threadIdx.x; e < cnt; e += kSoftThreads) plist[0][e] = (uint16_t)e;
  if (threadIdx.x == 0) { s_npend[0] = cnt; s_npend[1] = 0; }
  __syncthreads();
  int round = 0, cur_list = 0;
  for (;; ++round) {
    const uint16_t* pl = plist[cur_list];
    const int npend = s_npend[cur_list];
    // A: exact tentative scores of pending boxes with an overlapping neighbour finalized in the
    //    previous round: s0 times the factors of the final overlapping neighbours, in the
    //    reference's selection order (collected and insertion-sorted by (key, slot))
    if (round > 0) {
      for (int t = threadIdx.x; t < npend; t += kSoftThreads) {
        const int j = pl[t];
        const int32_t jx = F.sx[j], jy = F.sy[j], jz = F.sz[j];
        constexpr int kMaxNb = 24;
        // sorted (key, slot) list of the final overlapping neighbours; entries [0, nn) are
        // always written before they are read (insertion sort)
#pragma nv_diag_suppress 549
        uint64_t nk[kMaxNb];
        int nb[kMaxNb];
        int nn = 0;
        bool fresh = false;
        F.for_candidates(j, [&](int b) {
          if (F.state[b] != kSoftFinal || !soft_overlap(F.small, jx, jy, jz, F.sx[b], F.sy[b], F.sz[b])) return;
          fresh |= F.fround[b] == round - 1;
          if (nn <= kMaxNb) {
            if (nn < kMaxNb) {
              const uint64_t kb = F.fkey[b];
              int i = nn;
              while (i > 0 && soft_before(kb, b, nk[i - 1], nb[i - 1])) { nk[i] = nk[i - 1]; nb[i] = nb[i - 1]; --i; }
              nk[i] = kb; nb[i] = b;
            }
            ++nn;
          }
        });
#pragma nv_diag_default 549
        if (!fresh) continue;
        double tv = F.s0[j];
        if (nn <= kMaxNb) {
          for (int i = 0; i < nn; ++i)
            tv = soft_apply(F.small, tv, jx, jy, jz, F.sx[nb[i]], F.sy[nb[i]], F.sz[nb[i]], mode, theta, sigma);
        } else {  // many final neighbours (crowds): repeated minimum in key order
          uint64_t lk = 0;
          int li = -1;
          for (;;) {
            uint64_t bk = ~0ull;
            int bi = 0x7FFFFFFF;
            F.for_candidates(j, [&](int b) {
              if (F.state[b] != kSoftFinal) return;
              const uint64_t kb = F.fkey[b];
              if (!soft_before(lk, li, kb, b) || !soft_before(kb, b, bk, bi)) return;
              if (!soft_overlap(F.small, jx, jy, jz, F.sx[b], F.sy[b], F.sz[b])) return;
              bk = kb; bi = b;
            });
            if (bi == 0x7FFFFFFF) break;
            tv = soft_apply(F.small, tv, jx, jy, jz, F.sx[bi], F.sy[bi], F.sz[bi], mode, theta, sigma);
            lk = bk; li = bi;
          }
        }
        F.cur[j] = tv;
        F.fkey[j] = sort_key(tv);  // (read by others only once the box is final)
      }
    }
    __syncthreads();
    if (round >= kSoftMaxRounds) break;
    // B: a pending box that precedes every pending overlapping neighbour is final
    for (int t = threadIdx.x; t < npend; t += kSoftThreads) {
      const int j = pl[t];
      const int32_t jx = F.sx[j], jy = F.sy[j], jz = F.sz[j];
      const uint64_t kj = F.fkey[j];
      bool ready = true;
      F.for_candidates(j, [&](int n) {
        if (!ready || n == j || F.state[n] != kSoftPending) return;
        if (!soft_before(F.fkey[n], n, kj, j)) return;
        if (soft_overlap(F.small, jx, jy, jz, F.sx[n], F.sy[n], F.sz[n])) ready = false;
      });
      F.mark[j] = ready ? 1 : 0;
    }
    if (threadIdx.x == 0) s_npend[cur_list ^ 1] = 0;
    __syncthreads();
    // C: finalize (own slots only) and compact the still-pending boxes into the other list
    uint16_t* nl = plist[cur_list ^ 1];
    for (int base = 0; base < npend; base += kSoftThreads) {
      const int t = base + threadIdx.x;
      bool keep = false;
      int j = 0;
      if (t < npend) {
        j = pl[t];
        if (F.mark[j]) {
          F.fround[j] = (uint16_t)round;
          F.state[j] = kSoftFinal;
          F.mark[j] = 0;
        } else {
          keep = true;
        }
      }
      const unsigned bal = __ballot_sync(0xFFFFFFFFu, keep);
      int wbase = 0;
      if ((threadIdx.x & 31) == 0 && bal) wbase = atomicAdd(&s_npend[cur_list ^ 1], __popc(bal));
      wbase = __shfl_sync(0xFFFFFFFFu, wbase, 0);
      if (keep) nl[wbase + __popc(bal & lanemask_lt())] = (uint16_t)j;
    }
    __syncthreads();
    cur_list ^= 1;
    if (s_npend[cur_list] == 0) break;
  }
  // ---- dense crowds: finish with the reference's loop (cur is exact for every pending box)
  if (round >= kSoftMaxRounds) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (;;) {
      // argmin over pending of (sort key, index): pack (key >> 12 is not exact) -> two passes
      uint64_t bk = ~0ull;
      int bi = 0x7FFFFFFF;
      for (int j = threadIdx.x; j < cnt; j += kSoftThreads) {
        if (F.state[j] == kSoftFinal) continue;
        const uint64_t kj = sort_key(F.cur[j]);
        if (soft_before(kj, j, bk, bi)) { bk = kj; bi = j; }
      }
      for (int o = 16; o; o >>= 1) {
        const uint64_t ok = __shfl_xor_sync(0xFFFFFFFFu, bk, o);
        const int oi = __shfl_xor_sync(0xFFFFFFFFu, bi, o);
        if (soft_before(ok, oi, bk, bi)) { bk = ok; bi = oi; }
      }
      if (lane == 0) { s_best[warp] = bk; scan_tmp[warp] = (uint32_t)bi; }
      __syncthreads();
      if (warp == 0) {
        bk = lane < kSoftThreads / 32 ? s_best[lane] : ~0ull;
        bi = lane < kSoftThreads / 32 ? (int)scan_tmp[lane] : 0x7FFFFFFF;
        for (int o = 16; o; o >>= 1) {
          const uint64_t ok = __shfl_xor_sync(0xFFFFFFFFu, bk, o);
          const int oi = __shfl_xor_sync(0xFFFFFFFFu, bi, o);
          if (soft_before(ok, oi, bk, bi)) { bk = ok; bi = oi; }
        }
        if (lane == 0) s_stat[9] = bi;
      }
      __syncthreads();
      const int b = s_stat[9];
      if (b == 0x7FFFFFFF) break;
      const int32_t bx = F.sx[b], by = F.sy[b], bz = F.sz[b];
      for (int j = threadIdx.x; j < cnt; j += kSoftThreads) {
        if (j == b || F.state[j] == kSoftFinal) continue;
        F.cur[j] = soft_apply(F.small, F.cur[j], F.sx[j], F.sy[j], F.sz[j], bx, by, bz, mode, theta, sigma);
      }
      if (threadIdx.x == 0) F.state[b] = kSoftFinal;
      __syncthreads();
    }
  }
  // ---- rescored scores, input order
  for (int e = threadIdx.x; e < a.n_max; e += kSoftThreads) a.out_s[fbase + e] = e < cnt ? F.cur[e] : 0.0;
  if (threadIdx.x == 0) {
    a.status[f] = 0;
    if (a.rounds) a.rounds[f] = round;
  }
}

}  // namespace pnms

// pnms_greedy.cuh — classic greedy NMS (oracles.greedy_nms, oracles.py:64-85) on the device.
//
// Reference semantics: visit the valid detections by (score desc, index asc); a detection is
// kept unless an already-kept detection covers it, covers(cand, ref) requiring positive
// extents on both axes and w*h >= theta*(z_ref+1)^2 (oracles.py:20-29).  Unlike the engine's
// row AND, a suppressed box no longer suppresses (the chain fixture, workload.py:252-266,
// keeps {a, c} here and {a} in the engine).
//
// Parallel exact resolution: kept(j) <=> no kept higher-ranked box covers j.  Every round,
// each undecided box looks at its higher-ranked coverers: one kept -> removed; all removed
// (or none) -> kept; otherwise it waits.  Decisions are final and correct when made, each
// round decides at least the highest-ranked undecided box, so the loop ends after as many
// rounds as the longest suppression chain (a handful on detector output).
//
// Candidates: greedy never covers on zero overlap, so spatial cells are exact for every theta,
// and a coverer's corner lies within the theta reach of pnms_binned2.cuh (L left / up,
// z + 1 - R right / down, from w >= max(1, ceil(T_ref / (z_ref+1)))); frames with negative
// coordinates or a crowded cell scan all slots instead.  One CTA per frame; covers() is
// evaluated in exact 64-bit integer arithmetic against ceil(fl64(theta*a)).  The per-slot
// state of frames up to kGreedyMaxSlots lives in shared memory; larger frames (up to
// PNMS_MAX_SLOTS) keep the same layout in a caller-provided global workspace slice (L2-resident:
// ~46 B per slot), with the same code (GLOBAL template parameter).
#pragma once
#include "pnms_common.cuh"
#include "pnms_sort.cuh"
#include "pnms_binned.cuh"  // qdiv / div_magic

namespace pnms {

constexpr int kGreedyThreads = 512;
constexpr int kGreedyMaxSlots = 4096;   // largest frame whose state fits shared memory
constexpr int kGreedyCellMax = 64;
constexpr int kGreedyMaxCells = 65535;  // cell ids are 16-bit

enum GreedyState : uint8_t { kUndecided = 0, kKept = 1, kRemoved = 2 };

struct GreedyArgs {
  const int32_t *x, *y, *z;
  const double* s;
  const int32_t* counts;
  int batch, n_max, W32;
  double theta;
  int32_t* keep_idx;
  int32_t* keep_count;
  uint32_t* keep_mask;
  unsigned char* scratch;  // GLOBAL: [batch] slices of scratch_stride bytes (greedy_smem_bytes)
  size_t scratch_stride;
};

__host__ __device__ inline int greedy_npad(int n_max) { return (n_max + 127) & ~127; }
inline size_t greedy_smem_bytes(int n_max) {
  const size_t n = (size_t)greedy_npad(n_max);
  const size_t cells = n < 32 ? 64 : 2 * n;  // rectangular cells: up to two per box
  return (n * (4 * 3 + 8 + 8 + 1 + 1 + 2 + 2 + 2 + 2) + (cells + 4) * 4 + (n / 32 + 4) * 4 + 64 * 4 + 64 + 255) / 256 * 256;
}
__host__ __device__ inline int greedy_max_cells(int npad) {
  const int c = npad < 32 ? 64 : 2 * npad;
  return c > kGreedyMaxCells ? kGreedyMaxCells : c;
}

// covers(cand, ref) of oracles.py:20-29 in exact integer arithmetic; T = ceil(fl64(theta*a))
__device__ __forceinline__ bool greedy_covers(int32_t cx, int32_t cy, int32_t cz, int32_t rx, int32_t ry, int32_t rz,
                                              unsigned long long T) {
  const long long w = min((long long)cx + cz, (long long)rx + rz) - (long long)max(cx, rx) + 1;
  if (w <= 0) return false;
  const long long h = min((long long)cy + cz, (long long)ry + rz) - (long long)max(cy, ry) + 1;
  if (h <= 0) return false;
  return (unsigned long long)w * (unsigned long long)h >= T;
}

// the same in 32 bits, for frames whose x + z, y + z stay below 2^31 and whose sides are below
// 2^16 - 1 (extents, product and T then all fit; every BASELINE frame)
__device__ __forceinline__ bool greedy_covers32(int32_t cx, int32_t cy, int32_t cz, int32_t rx, int32_t ry, int32_t rz,
                                                uint32_t T) {
  const int w = min(cx + cz, rx + rz) - max(cx, rx) + 1;
  const int h = min(cy + cz, ry + rz) - max(cy, ry) + 1;
  return (w > 0) & (h > 0) && (uint32_t)w * (uint32_t)h >= T;
}

__device__ __forceinline__ unsigned long long greedy_threshold(double theta, int32_t z) {
  // Python: theta * ((z+1)*(z+1)) converts the exact integer area to float64, then multiplies
  const long long a = ((long long)z + 1) * ((long long)z + 1);
  const double thr = __dmul_rn(theta, __ll2double_rn(a));
  const double c = ceil(thr);
  return c >= 1.8e19 ? ~0ull : (unsigned long long)c;
}

template <bool GLOBAL>
__global__ void __launch_bounds__(kGreedyThreads) pnms_greedy_frame(GreedyArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ int s_stat[8];   // 0 minx 1 miny 2 maxx 3 maxy 4 maxz 5 bin_ok 6 big 7 undecided
  // the reach of a coverer (as pnms_binned2.cuh): ref i covers cand j only if w >= wmin_i =
  // max(1, ceil(T_i / (z_i+1))) (h <= z_i + 1), so x_i lies in [x_j - L, x_j + z_j + 1 - R] with
  // L = max_i (z_i + 1 - wmin_i), R = min_i wmin_i (same for y)
  __shared__ long long s_L, s_R;
  __shared__ int s_small;  // every cell coordinate below 2^16: one IMAD.HI per division
  __shared__ uint32_t scan_tmp[64];
  const int f = blockIdx.x;
  const long long fbase = (long long)f * a.n_max;
  const int cnt = frame_count(a.counts, f, a.n_max);
  const int npad = greedy_npad(a.n_max);
  const int max_cells = greedy_max_cells(npad);
  unsigned char* base;
  if constexpr (GLOBAL) base = a.scratch + (size_t)f * a.scratch_stride;
  else base = smem_raw;
  int32_t* sx = reinterpret_cast<int32_t*>(base);
  int32_t* sy = sx + npad;
  int32_t* sz = sy + npad;
  uint64_t* key = reinterpret_cast<uint64_t*>(sz + npad);
  unsigned long long* thr = reinterpret_cast<unsigned long long*>(key + npad);
  uint8_t* state = reinterpret_cast<uint8_t*>(thr + npad);
  uint8_t* dec = state + npad;  // this round's decisions, applied after a barrier (no read/write race)
  uint16_t* cellof = reinterpret_cast<uint16_t*>(dec + npad);
  uint16_t* list = cellof + npad;
  uint16_t* ulist[2] = {list + npad, list + 2 * npad};  // undecided boxes, double-buffered
  uint32_t* cstart = reinterpret_cast<uint32_t*>(list + 3 * npad);
  uint32_t* kbits = cstart + max_cells + 4;

  if (threadIdx.x == 0) {
    s_stat[0] = s_stat[1] = 0x7FFFFFFF;
    s_stat[2] = s_stat[3] = -0x7FFFFFFF;
    s_stat[4] = 0; s_stat[5] = 1; s_stat[6] = 0; s_stat[7] = 0;
    s_L = 0; s_R = 0x7FFFFFFFFFFFFFFFll; s_small = 0;
  }
  for (int w = threadIdx.x; w < npad / 32; w += kGreedyThreads) kbits[w] = 0u;
  __syncthreads();
  // ---- load
  for (int e = threadIdx.x; e < cnt; e += kGreedyThreads) {
    const long long g = fbase + e;
    const int32_t xv = a.x[g], yv = a.y[g], zv = a.z[g];
    const double sv = a.s[g];
    sx[e] = xv; sy[e] = yv; sz[e] = zv;
    key[e] = sort_key(sv);
    const unsigned long long T = greedy_threshold(a.theta, zv);
    thr[e] = T;
    if (zv >= 0 && sv == sv) {
      const unsigned long long zz = (unsigned long long)zv + 1ull;
      const unsigned long long q = T / zz + (T % zz != 0ull);
      const long long wmin = q < 1ull ? 1ll : (q > zz ? (long long)zz + 1 : (long long)q);  // > z+1: never covers
      atomicMax(&s_L, (long long)zz - wmin);
      atomicMin(&s_R, wmin);
    }
    state[e] = (sv != sv) ? kKept : kUndecided;  // NaN: unordered, never covers (documented)
    dec[e] = kUndecided;
    if (xv < 0 || yv < 0 || zv < 0) atomicAnd(&s_stat[5], 0);
    atomicMin(&s_stat[0], xv); atomicMin(&s_stat[1], yv);
    atomicMax(&s_stat[2], xv); atomicMax(&s_stat[3], yv); atomicMax(&s_stat[4], zv);
  }
  __syncthreads();
  // ---- spatial cells (exact for greedy at any theta: zero overlap never covers)
  bool bin = s_stat[5] != 0 && cnt > 0;
  // cells Sx wide and Sy tall (any shape is exact: a box's coverers have their corner in
  // [x - max_z, x + z] x [y - max_z, y + z]); narrow cells tighten the x range of a scan,
  // tall ones keep the cell rows per scan few (as in pnms_binned.cuh)
  int Sx = 1, Sy = 1, GX = 1, GY = 1;
  const int ox = s_stat[0], oy = s_stat[1];
  const long long L = max(s_L, 0ll), R = min(s_R, 0x7FFFFFFFll);
  if (bin) {
    Sy = (int)min(L + 1, (long long)s_stat[4] + 1);
    if (Sy <= 0) bin = false;  // z = INT_MAX
    Sx = max(Sy >> 2, 1);
  }
  if (bin) {
    for (;;) {
      GX = (int)(((long long)s_stat[2] - ox) / Sx + 1);
      GY = (int)(((long long)s_stat[3] - oy) / Sy + 1);
      if ((long long)GX * GY <= max_cells) break;
      if (Sy > (1 << 29)) { GX = GY = 1; break; }
      if (Sx < Sy) Sx *= 2;
      else { Sx *= 2; Sy *= 2; }
    }
    const int cells = GX * GY;
    if (threadIdx.x == 0)
      s_small = s_stat[2] - ox + (long long)s_stat[4] + 1 < 32768 && s_stat[3] - oy + (long long)s_stat[4] + 1 < 32768;
    for (int c = threadIdx.x; c <= cells; c += kGreedyThreads) cstart[c] = 0u;
    __syncthreads();
    for (int e = threadIdx.x; e < cnt; e += kGreedyThreads) {
      // (binned frames have non-negative coordinates: the offsets and quotients fit 32 bits)
      const int c = (int)((uint32_t)(sy[e] - oy) / (uint32_t)Sy) * GX + (int)((uint32_t)(sx[e] - ox) / (uint32_t)Sx);
      cellof[e] = (uint16_t)c;
      atomicAdd(&cstart[c], 1u);
    }
    __syncthreads();
    {
      const int per = (cells + 1 + kGreedyThreads - 1) / kGreedyThreads;
      const int b0 = threadIdx.x * per;
      uint32_t sum = 0, big = 0;
      for (int t = 0; t < per; ++t) {
        const int c = b0 + t;
        if (c < cells) { sum += cstart[c]; big = max(big, cstart[c]); }
      }
      big = __reduce_max_sync(0xFFFFFFFFu, big);
      if ((threadIdx.x & 31) == 0) atomicMax(&s_stat[6], (int)big);
      uint32_t run = block_exclusive_scan(sum, scan_tmp, nullptr);
      for (int t = 0; t < per; ++t) {
        const int c = b0 + t;
        if (c < cells) { const uint32_t v = cstart[c]; cstart[c] = run; run += v; }
      }
      if (threadIdx.x == 0) cstart[cells] = (uint32_t)cnt;
    }
    __syncthreads();
    bin = s_stat[6] <= kGreedyCellMax;
    if (bin) {
      // scatter with cstart as the cursor: afterwards cstart[c] = end(c) = start(c+1)
      for (int e = threadIdx.x; e < cnt; e += kGreedyThreads) {
        const uint32_t pos = atomicAdd(&cstart[cellof[e]], 1u);
        list[pos] = (uint16_t)e;
      }
    }
  }
  __syncthreads();
  // After the scatter, cstart[c] == end(c) == start(c+1); start(0) = 0.
  const bool small = bin && s_small;
  // 32-bit coverage tests (greedy_covers32): non-negative coordinates (bin), x + z and y + z
  // below 2^31, sides below 2^16 - 1
  const bool c32 = bin && (long long)s_stat[2] + s_stat[4] < 0x7FFFFFFFLL &&
                   (long long)s_stat[3] + s_stat[4] < 0x7FFFFFFFLL && s_stat[4] < 65534;
  const uint32_t Mx = div_magic(Sx), My = div_magic(Sy);
  // ---- rounds over a compacted list of the undecided boxes; decisions go to dec[] and are
  // applied after a barrier (every box's slots are written only by its own thread)
  __shared__ int s_nund[2];
  for (int e = threadIdx.x; e < cnt; e += kGreedyThreads) ulist[0][e] = (uint16_t)e;
  if (threadIdx.x == 0) { s_nund[0] = cnt; s_nund[1] = 0; }
  __syncthreads();
  for (int cur = 0;; cur ^= 1) {
    const uint16_t* ul = ulist[cur];
    const int nund = s_nund[cur];
    for (int t = threadIdx.x; t < nund; t += kGreedyThreads) {
      const int j = ul[t];
      if (state[j] != kUndecided) continue;  // NaN rows start kept
      const uint64_t kj = key[j];
      const int32_t jx = sx[j], jy = sy[j], jz = sz[j];
      bool kept_cov = false, undec_cov = false;
      if (bin) {
        // the cells the coverers' corners can lie in; one contiguous run per cell row
        const long long lx = max(0LL, (long long)jx - L - ox), ly = max(0LL, (long long)jy - L - oy);
        const long long hx = (long long)jx + jz + 1 - R - ox, hy = (long long)jy + jz + 1 - R - oy;
        int cx0, cy0, cx1, cy1;
        if (small) {  // (0 <= lx <= hx < 2^16 when hx >= 0)
          cx0 = Sx == 1 ? (int)lx : qdiv((int)lx, Mx); cy0 = Sy == 1 ? (int)ly : qdiv((int)ly, My);
          cx1 = Sx == 1 ? (int)hx : qdiv((int)max(hx, 0LL), Mx); cy1 = Sy == 1 ? (int)hy : qdiv((int)max(hy, 0LL), My);
        } else {
          cx0 = (int)(lx / Sx); cy0 = (int)(ly / Sy);
          cx1 = (int)(max(hx, 0LL) / Sx); cy1 = (int)(max(hy, 0LL) / Sy);
        }
        cx1 = min(GX - 1, cx1);
        // (hx or hy < 0: no ref reaches j — an empty range, so j is kept below)
        cy1 = hx < 0 || hy < 0 ? cy0 - 1 : min(GY - 1, cy1);
        for (int yy = cy0; yy <= cy1 && !kept_cov; ++yy) {
          const int c0 = yy * GX + cx0, c1 = yy * GX + cx1;
          const int b = c0 == 0 ? 0 : (int)cstart[c0 - 1], en = (int)cstart[c1];
          for (int q = b; q < en; ++q) {
            const int i = list[q];
            const uint8_t si = state[i];
            if (si == kRemoved) continue;
            const uint64_t ki = key[i];
            if (!(ki < kj || (ki == kj && i < j))) continue;
            if (c32 ? !greedy_covers32(jx, jy, jz, sx[i], sy[i], sz[i], (uint32_t)thr[i])
                    : !greedy_covers(jx, jy, jz, sx[i], sy[i], sz[i], thr[i]))
              continue;
            if (si == kKept) { kept_cov = true; break; }
            undec_cov = true;
          }
        }
      } else {
        for (int i = 0; i < cnt; ++i) {
          const uint8_t si = state[i];
          if (si == kRemoved) continue;
          const uint64_t ki = key[i];
          if (!(ki < kj || (ki == kj && i < j))) continue;
          if (!greedy_covers(jx, jy, jz, sx[i], sy[i], sz[i], thr[i])) continue;
          if (si == kKept) { kept_cov = true; break; }
          undec_cov = true;
        }
      }
      if (kept_cov) dec[j] = kRemoved;
      else if (!undec_cov) dec[j] = kKept;
    }
    if (threadIdx.x == 0) s_nund[cur ^ 1] = 0;
    __syncthreads();
    uint16_t* nl = ulist[cur ^ 1];
    for (int base = 0; base < nund; base += kGreedyThreads) {
      const int t = base + threadIdx.x;
      bool keep = false;
      int j = 0;
      if (t < nund) {
        j = ul[t];
        if (dec[j] != kUndecided) { state[j] = dec[j]; dec[j] = kUndecided; }
        keep = state[j] == kUndecided;
      }
      const unsigned bal = __ballot_sync(0xFFFFFFFFu, keep);
      int wbase = 0;
      if ((threadIdx.x & 31) == 0 && bal) wbase = atomicAdd(&s_nund[cur ^ 1], __popc(bal));
      wbase = __shfl_sync(0xFFFFFFFFu, wbase, 0);
      if (keep) nl[wbase + __popc(bal & lanemask_lt())] = (uint16_t)j;
    }
    __syncthreads();
    if (s_nund[cur ^ 1] == 0) break;
  }
  // ---- compaction of the kept boxes (ascending input order, oracles.py:84)
  for (int j = threadIdx.x; j < cnt; j += kGreedyThreads)
    if (state[j] == kKept) atomicOr(&kbits[j >> 5], 1u << (j & 31));
  __syncthreads();
  const int wpt = (a.W32 + kGreedyThreads - 1) / kGreedyThreads;
  const int w0 = threadIdx.x * wpt, w1 = min(w0 + wpt, a.W32);
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
  if (threadIdx.x == 0 && a.keep_count) a.keep_count[f] = (int32_t)total;
}

}  // namespace pnms

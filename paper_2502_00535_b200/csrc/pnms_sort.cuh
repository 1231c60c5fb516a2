// pnms_sort.cuh — per-frame preparation and segmented score sort.
//
// The reference never sorts: it tests all d_max^2 ordered
// slot pairs and lets the score gate `s_i < s_j` (engine.py:233-235) discard half of them.
// Sorting every frame by (score desc, index asc) turns that gate into a loop bound: sorted
// row p only needs columns q < lim[p], where
//   lim[p] = first position of p's equal-score group   (tie_break = paper_faithful)
//   lim[p] = p                                         (tie_break = by_index)
// which is exactly the set of slots that pass the reference's gate.  The sort is a stable
// LSD radix sort on the 64-bit order-preserving key, so equal scores keep input order.
//
// Frames of up to kSortMax slots are sorted inside one CTA (pnms_prep_sort_frame).  Larger
// frames are cut into kSortMax-slot chunks sorted independently (pnms_prep_sort_chunk) and
// merged by rank (pnms_merge_rank): a slot's global position is its position in its own
// chunk plus, for every other chunk, the number of slots there that precede it — found by a
// binary search, because chunks cover contiguous index ranges.
#pragma once
#include "pnms_common.cuh"

namespace pnms {

struct PrepArgs {
  const int32_t* x;
  const int32_t* y;
  const int32_t* z;
  const double* s;
  const int32_t* counts;  // may be null
  int batch, n_max, npad, tie_break, W32, nchunks;
  double theta;
  uint8_t* rec;       // [batch][n_max] records, kRecBytes stride per frame slot
  int32_t* perm;      // [batch][n_max] sorted position -> input index
  int32_t* lim;       // [batch][n_max] column limit of the sorted row
  uint32_t* supp;     // [batch][W32]  suppression bits in sorted order (zeroed here)
  FrameMeta* meta;    // [batch]
  uint64_t* sk_scratch;   // chunk mode: sorted keys   [batch][n_max]
  int32_t* idx_scratch;   // chunk mode: sorted index  [batch][n_max]
  const uint8_t* dense;   // optional [batch]: process frame f only if dense[f] != 0
  const int32_t* list;    // optional: process only frames list[0 .. *list_count) (grid-stride)
  const int* list_count;
};

__device__ __forceinline__ bool frame_skipped(const uint8_t* dense, int f) { return dense && !dense[f]; }

__device__ __forceinline__ int frame_count(const int32_t* counts, int f, int n_max) {
  int c = counts ? counts[f] : n_max;
  return c < 0 ? 0 : (c > n_max ? n_max : c);
}

// lower_bound / upper_bound over an ascending array
__device__ __forceinline__ int lower_bound_u64(const uint64_t* a, int n, uint64_t v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ int upper_bound_u64(const uint64_t* a, int n, uint64_t v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (a[mid] <= v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// Stable block sort (ascending) of npad = 512*E (key, idx) pairs held in shared memory.
//  1. LSD radix passes with 8-bit digits over the HIGH 32 bits of the key only; digits on
//     which every key agrees (diff_hi == 0 there) are skipped — for scores in [0.05, 1) the
//     top byte is constant, so three passes run.  Warp w owns the contiguous run
//     [w*32E, (w+1)*32E); inside a warp, rounds of 32 consecutive slots are ranked by a
//     ballot multisplit (8 ballots) so the scatter preserves input order.  Per-warp digit
//     counters live at hist[w*256 + d] (conflict-free for distinct digits).
//  2. Runs of equal high words (rare: ~1 per 2048 random scores) are re-ranked exactly by
//     (full key, idx) by counting inside the run; NaN keys and padding are left as they are
//     (their order never matters: they are never columns of an active row).
// On return *k / *id point at the sorted sequence of the first `cnt` slots.
__device__ void block_sort_keys(uint64_t** k, uint16_t** id, uint64_t* k2, uint16_t* id2, uint32_t* hist,
                                uint32_t* scan_tmp, int E, int cnt, uint32_t diff_hi) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t lt = lanemask_lt();
  uint64_t* ka = *k;
  uint16_t* ia = *id;
  uint64_t* kb = k2;
  uint16_t* ib = id2;
  const int wbase = warp * 32 * E;
  uint32_t* whist = hist + warp * 256;
  for (int sh = 0; sh < 32; sh += 8) {
    if (((diff_hi >> sh) & 0xFFu) == 0) continue;
    for (int i = threadIdx.x; i < 256 * kSortWarps; i += kSortThreads) hist[i] = 0;
    __syncthreads();
    uint64_t key[8];
    uint16_t ix[8];
    uint32_t dig[8], peers[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if (r < E) {
        const int e = wbase + r * 32 + lane;
        key[r] = ka[e];
        ix[r] = ia[e];
        const uint32_t d = (uint32_t)(key[r] >> (32 + sh)) & 0xFFu;
        uint32_t pm = 0xFFFFFFFFu;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          const uint32_t bal = __ballot_sync(0xFFFFFFFFu, (d >> b) & 1u);
          pm &= ((d >> b) & 1u) ? bal : ~bal;
        }
        dig[r] = d;
        peers[r] = pm;
        if (lane == __ffs(pm) - 1) whist[d] += __popc(pm);
        __syncwarp();
      }
    }
    __syncthreads();
    // digit-major exclusive offsets: base(d) + sum of warps before w for digit d
    {
      uint32_t tot = 0;
      if (threadIdx.x < 256) {
        for (int w = 0; w < kSortWarps; ++w) {
          const uint32_t v = hist[w * 256 + threadIdx.x];
          hist[w * 256 + threadIdx.x] = tot;
          tot += v;
        }
      }
      const uint32_t base = block_exclusive_scan(threadIdx.x < 256 ? tot : 0u, scan_tmp, nullptr);
      if (threadIdx.x < 256)
        for (int w = 0; w < kSortWarps; ++w) hist[w * 256 + threadIdx.x] += base;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if (r < E) {
        const uint32_t b0 = whist[dig[r]];
        const uint32_t pos = b0 + __popc(peers[r] & lt);
        kb[pos] = key[r];
        ib[pos] = ix[r];
        __syncwarp();
        if (lane == __ffs(peers[r]) - 1) whist[dig[r]] = b0 + __popc(peers[r]);
        __syncwarp();
      }
    }
    __syncthreads();
    uint64_t* tk = ka; ka = kb; kb = tk;
    uint16_t* ti = ia; ia = ib; ib = ti;
  }
  // exact fix-up of equal-high-word runs
  for (int p = threadIdx.x; p < cnt; p += kSortThreads) {
    const uint64_t sk = ka[p];
    const uint32_t h = (uint32_t)(sk >> 32);
    const bool run = sk != kNanSortKey && ((p > 0 && (uint32_t)(ka[p - 1] >> 32) == h) ||
                                           (p + 1 < cnt && (uint32_t)(ka[p + 1] >> 32) == h));
    int dst = p;
    if (run) {
      int rs = p, re = p + 1;
      while (rs > 0 && (uint32_t)(ka[rs - 1] >> 32) == h) --rs;
      while (re < cnt && (uint32_t)(ka[re] >> 32) == h) ++re;
      const uint16_t me = ia[p];
      int rank = 0;
      for (int q = rs; q < re; ++q) {
        const uint64_t o = ka[q];
        rank += (o < sk) || (o == sk && ia[q] < me);
      }
      dst = rs + rank;
    }
    kb[dst] = sk;
    ib[dst] = ia[p];
  }
  __syncthreads();
  *k = kb;
  *id = ib;
}

// u64 warp reductions (no native 64-bit redux)
__device__ __forceinline__ uint64_t warp_min_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const uint64_t t = __shfl_xor_sync(0xFFFFFFFFu, v, o);
    v = t < v ? t : v;
  }
  return v;
}
__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const uint64_t t = __shfl_xor_sync(0xFFFFFFFFu, v, o);
    v = t > v ? t : v;
  }
  return v;
}

constexpr int kBucketMaxLoad = 64;  // larger buckets fall back to the radix sort

// Bucket sort with exact in-bucket ranking.  Keys of the non-NaN slots are mapped linearly
// onto nb buckets over [kmin, kmax] (monotone, so a higher bucket always holds strictly
// larger keys); one counting pass places every slot in its bucket, then each slot finds its
// exact position inside the bucket by counting the members that precede it in
// (key, index) order.  Valid NaN slots go to bucket nb and padding slots (e >= cnt) to
// bucket nb+1, so NaN rows occupy [n_active, cnt) and padding stays past cnt; the internal
// order of those two buckets is irrelevant.  Returns false (input untouched) when a real
// bucket holds more than kBucketMaxLoad slots — the caller then runs block_sort_keys.
// scratch: cnt_s needs nb + 2 words, off_s nb + 3 words.
// Inverse of sort_key for non-NaN keys (canonical +0.0 for zero).
__device__ __forceinline__ double key_to_score(uint64_t sk) {
  const uint64_t key = ~sk;
  const uint64_t b = (key >> 63) ? (key & 0x7FFFFFFFFFFFFFFFull) : ~key;
  return __longlong_as_double((long long)b);
}

// Bucket of a slot.  With a finite score range the buckets split [smax, smin] linearly in
// score VALUE (ascending sort key = descending score); otherwise linearly in key bits.
// Both maps are monotone non-decreasing in the key, which is all exactness needs.
struct BucketMap {
  uint64_t kmin;
  int shift;       // key-bit map
  double smax, scale;  // value map (scale <= 0: use the key-bit map)
  int nb;
  __device__ __forceinline__ int operator()(uint64_t sk, int e, int cnt) const {
    if (e >= cnt) return nb + 1;
    if (sk == kNanSortKey) return nb;
    if (scale > 0.0) {
      const double t = __dmul_rn(__dsub_rn(smax, key_to_score(sk)), scale);
      return min(nb - 1, (int)t);
    }
    return (int)((sk - kmin) >> shift);
  }
};

__device__ bool block_bucket_sort(uint64_t** k, uint16_t** id, uint64_t* k2, uint16_t* id2, uint32_t* cnt_s,
                                  uint32_t* off_s, uint32_t* scan_tmp, int npad, int cnt, uint64_t kmin,
                                  uint64_t kmax, int nb) {
  uint64_t* ka = *k;
  uint16_t* ia = *id;
  BucketMap bm;
  bm.nb = nb;
  bm.kmin = kmin;
  {
    const uint64_t range = kmax - kmin;
    const int bits = range ? 64 - __clzll((long long)range) : 0;  // bits needed for the range
    const int nb_bits = 31 - __clz(nb);
    bm.shift = bits > nb_bits ? bits - nb_bits : 0;
    const double smax = key_to_score(kmin), smin = key_to_score(kmax);
    const double span = smax - smin;
    bm.smax = smax;
    bm.scale = (isfinite(smax) && isfinite(smin) && span > 0.0 && isfinite(span)) ? (double)nb / span : -1.0;
  }
  const int nbk = nb + 2;  // real buckets + NaN bucket + padding bucket
  for (int b = threadIdx.x; b < nbk; b += kSortThreads) cnt_s[b] = 0u;
  __syncthreads();
  for (int e = threadIdx.x; e < npad; e += kSortThreads) atomicAdd(&cnt_s[bm(ka[e], e, cnt)], 1u);
  __syncthreads();
  // exclusive scan of the counts; also the largest real bucket
  const int per = (nbk + kSortThreads - 1) / kSortThreads;
  const int b0 = threadIdx.x * per;
  uint32_t sum = 0, big = 0;
  for (int t = 0; t < per; ++t) {
    const int b = b0 + t;
    if (b < nbk) {
      sum += cnt_s[b];
      if (b < nb) big = max(big, cnt_s[b]);
    }
  }
  big = __reduce_max_sync(0xFFFFFFFFu, big);
  uint32_t total;
  uint32_t run = block_exclusive_scan(sum, scan_tmp, &total);
  if ((threadIdx.x & 31) == 0) atomicMax(&scan_tmp[40], big);
  for (int t = 0; t < per; ++t) {
    const int b = b0 + t;
    if (b < nbk) {
      off_s[b] = run;
      run += cnt_s[b];
    }
  }
  if (threadIdx.x == 0) off_s[nbk] = npad;
  __syncthreads();
  const bool ok = scan_tmp[40] <= (uint32_t)kBucketMaxLoad;
  __syncthreads();
  if (threadIdx.x == 0) scan_tmp[40] = 0u;
  if (!ok) return false;
  // scatter (cnt_s becomes the insertion cursor)
  for (int b = threadIdx.x; b < nbk; b += kSortThreads) cnt_s[b] = off_s[b];
  __syncthreads();
  for (int e = threadIdx.x; e < npad; e += kSortThreads) {
    const uint64_t sk = ka[e];
    const uint32_t pos = atomicAdd(&cnt_s[bm(sk, e, cnt)], 1u);
    k2[pos] = sk;
    id2[pos] = ia[e];
  }
  __syncthreads();
  // exact rank inside each real bucket -> final position (written back into ka/ia)
  for (int p = threadIdx.x; p < npad; p += kSortThreads) {
    const uint64_t sk = k2[p];
    const uint16_t me = id2[p];
    int dst = p;
    if (p < cnt && sk != kNanSortKey) {
      const int b = bm(sk, 0, 1);
      const int bs = (int)off_s[b], be = (int)off_s[b + 1];
      int rank = 0;
      for (int q = bs; q < be; ++q) {
        const uint64_t o = k2[q];
        rank += (o < sk) || (o == sk && id2[q] < me);
      }
      dst = bs + rank;
    }
    ka[dst] = sk;
    ia[dst] = me;
  }
  __syncthreads();
  return true;
}

__device__ __forceinline__ void write_record(uint8_t* rec_frame, int pos, int mode, int32_t x, int32_t y,
                                             int32_t z, double theta) {
  if (mode == kWide) {
    reinterpret_cast<RecWide*>(rec_frame)[pos] = make_rec_wide(x, y, z, theta);
  } else {
    reinterpret_cast<RecNarrow*>(rec_frame)[pos] = make_rec_narrow(x, y, z, theta, mode);
  }
}

struct __align__(16) LoadStats {
  unsigned long long kmin, kmax;   // range of the non-NaN sort keys
  uint32_t or_lo, or_hi, and_lo, and_hi;
  int mode, n_act, neg, pos, zero;
};

// Loads slots [e0, e0+len) of a frame into (key, local idx) smem arrays of size npad and
// reduces the statistics the later phases need.  Slots past len are padded with the NaN
// key (they sort last, after real NaNs, by stability).
__device__ void load_keys(const PrepArgs& a, long long fbase, int e0, int len, int npad, uint64_t* k,
                          uint16_t* id, LoadStats* st, int32_t* sx = nullptr, int32_t* sy = nullptr,
                          int32_t* sz = nullptr) {
  const int lane = threadIdx.x & 31;
  uint32_t or_lo = 0, or_hi = 0, and_lo = ~0u, and_hi = ~0u;
  uint64_t kmin = ~0ull, kmax = 0ull;
  int mode = kNarrow7, n_act = 0, neg = 0, pos = 0, zero = 0;
  for (int e = threadIdx.x; e < npad; e += kSortThreads) {
    uint64_t key = kNanSortKey;
    if (e < len) {
      long long g = fbase + e0 + e;
      double sv = a.s[g];
      key = sort_key(sv);
      const int32_t xv = a.x[g], yv = a.y[g], zv = a.z[g];
      if (sx) { sx[e] = xv; sy[e] = yv; sz[e] = zv; }
      int m = frame_mode_of(xv, yv, zv);
      mode = m > mode ? m : mode;
      or_lo |= (uint32_t)key; or_hi |= (uint32_t)(key >> 32);
      and_lo &= (uint32_t)key; and_hi &= (uint32_t)(key >> 32);
      n_act += (key != kNanSortKey);
      if (key != kNanSortKey) {
        kmin = key < kmin ? key : kmin;
        kmax = key > kmax ? key : kmax;
      }
      neg += (sv < 0.0);
      pos += (sv > 0.0);
      zero += (sv == 0.0);
    }
    k[e] = key;
    id[e] = static_cast<uint16_t>(e);
  }
  or_lo = __reduce_or_sync(0xFFFFFFFFu, or_lo);
  or_hi = __reduce_or_sync(0xFFFFFFFFu, or_hi);
  and_lo = __reduce_and_sync(0xFFFFFFFFu, and_lo);
  and_hi = __reduce_and_sync(0xFFFFFFFFu, and_hi);
  mode = __reduce_max_sync(0xFFFFFFFFu, mode);
  n_act = __reduce_add_sync(0xFFFFFFFFu, n_act);
  neg = __reduce_add_sync(0xFFFFFFFFu, neg);
  pos = __reduce_add_sync(0xFFFFFFFFu, pos);
  zero = __reduce_add_sync(0xFFFFFFFFu, zero);
  kmin = warp_min_u64(kmin);
  kmax = warp_max_u64(kmax);
  if (lane == 0) {
    atomicMin(&st->kmin, (unsigned long long)kmin);
    atomicMax(&st->kmax, (unsigned long long)kmax);
    atomicOr(&st->or_lo, or_lo); atomicOr(&st->or_hi, or_hi);
    atomicAnd(&st->and_lo, and_lo); atomicAnd(&st->and_hi, and_hi);
    atomicMax(&st->mode, mode);
    atomicAdd(&st->n_act, n_act); atomicAdd(&st->neg, neg);
    atomicAdd(&st->pos, pos); atomicAdd(&st->zero, zero);
  }
}

// Shared-memory carve-up for both sort kernels.
struct SortSmem {
  uint64_t *ka, *kb;
  uint16_t *ia, *ib;
  int32_t *sx, *sy, *sz;   // staged coordinates (frame kernel only)
  uint32_t* hist;
  uint32_t* scan_tmp;
  LoadStats* st;
  unsigned long long* lim_acc;
};
__device__ __forceinline__ SortSmem carve_sort_smem(unsigned char* base, int npad) {
  SortSmem m;
  m.ka = reinterpret_cast<uint64_t*>(base);
  m.kb = m.ka + npad;
  m.hist = reinterpret_cast<uint32_t*>(m.kb + npad);
  m.scan_tmp = m.hist + 256 * kSortWarps + 64;  // hist has 64 spare words for the bucket offsets
  m.st = reinterpret_cast<LoadStats*>(m.scan_tmp + 64);
  m.lim_acc = reinterpret_cast<unsigned long long*>(m.st + 1);  // LoadStats is 16-byte aligned
  m.ia = reinterpret_cast<uint16_t*>(m.lim_acc + 2);
  m.ib = m.ia + npad;
  m.sx = reinterpret_cast<int32_t*>(m.ib + npad);
  m.sy = m.sx + npad;
  m.sz = m.sy + npad;
  return m;
}
inline size_t sort_smem_bytes(int npad) {
  static_assert(sizeof(LoadStats) % 16 == 0, "keeps lim_acc 8-byte aligned");
  return (size_t)npad * 16 + (256 * kSortWarps + 64) * 4 + 64 * 4 + sizeof(LoadStats) + 16 + (size_t)npad * 4;
}
inline size_t sort_frame_smem_bytes(int npad) {
  return sort_smem_bytes(npad) + (size_t)npad * 12;
}

__device__ __forceinline__ void init_stats(LoadStats* st, unsigned long long* lim_acc) {
  if (threadIdx.x == 0) {
    st->kmin = ~0ull;
    st->kmax = 0ull;
    st->or_lo = st->or_hi = 0;
    st->and_lo = st->and_hi = ~0u;
    st->mode = kNarrow7;
    st->n_act = st->neg = st->pos = st->zero = 0;
    *lim_acc = 0ull;
  }
}

// One CTA per frame (n_max <= kSortMax): load, sort, derive limits, emit sorted records.
__device__ __forceinline__ void prep_sort_frame_body(const PrepArgs& a, int f, unsigned char* smem_raw) {
  const long long fbase = (long long)f * a.n_max;
  const int cnt = frame_count(a.counts, f, a.n_max);
  SortSmem m = carve_sort_smem(smem_raw, a.npad);
  init_stats(m.st, m.lim_acc);
  if (threadIdx.x == 0) m.scan_tmp[40] = 0u;
  __syncthreads();
  load_keys(a, fbase, 0, cnt, a.npad, m.ka, m.ia, m.st, m.sx, m.sy, m.sz);
  __syncthreads();
  const uint32_t diff_hi = m.st->or_hi ^ m.st->and_hi;
  const int mode = m.st->mode;
  const int n_act = m.st->n_act;
  uint64_t* k = m.ka;
  uint16_t* id = m.ia;
  bool sorted = cnt <= 1;
  if (!sorted && n_act > 0) {
    const int nb = a.npad >= 4096 ? 2048 : (a.npad >= 2048 ? 2048 : a.npad);
    sorted = block_bucket_sort(&k, &id, m.kb, m.ib, m.hist, m.hist + 2052, m.scan_tmp, a.npad, cnt, m.st->kmin,
                               m.st->kmax, nb);
  }
  if (!sorted) block_sort_keys(&k, &id, m.kb, m.ib, m.hist, m.scan_tmp, a.npad / kSortThreads, cnt, diff_hi);

  uint8_t* rec_frame = a.rec + fbase * kRecBytes;
  unsigned long long lsum = 0;
  // thread t owns sorted positions [t*E, t*E+E); tie-group starts by a block max-scan
  const int E = a.npad / kSortThreads;
  const int pb = threadIdx.x * E;
  int run = -1;
  for (int t = 0; t < E; ++t) {
    const int p = pb + t;
    if (p < n_act && (p == 0 || k[p] != k[p - 1])) run = p;
  }
  const int carry = block_exclusive_max_scan(run, reinterpret_cast<int*>(m.scan_tmp));
  run = carry;
  for (int t = 0; t < E; ++t) {
    const int p = pb + t;
    if (p >= cnt) break;
    if (p < n_act && (p == 0 || k[p] != k[p - 1])) run = p;
    const int l = (p < n_act) ? ((a.tie_break == 1) ? p : run) : 0;
    lsum += (unsigned long long)l;
    const int i = id[p];
    a.perm[fbase + p] = i;
    a.lim[fbase + p] = l;
    write_record(rec_frame, p, mode, m.sx[i], m.sy[i], m.sz[i], a.theta);
  }
  for (int w = threadIdx.x; w < a.W32; w += kSortThreads) a.supp[(long long)f * a.W32 + w] = 0u;
  lsum = __reduce_add_sync(0xFFFFFFFFu, (unsigned)(lsum & 0xFFFFFFFFull)) +
         ((unsigned long long)__reduce_add_sync(0xFFFFFFFFu, (unsigned)(lsum >> 32)) << 32);
  if ((threadIdx.x & 31) == 0) atomicAdd(m.lim_acc, lsum);
  __syncthreads();
  if (threadIdx.x == 0) {
    FrameMeta fm;
    fm.n_active = n_act;
    fm.mode = mode;
    fm.cnt_neg = m.st->neg;
    fm.cnt_pos = m.st->pos;
    fm.cnt_zero = m.st->zero;
    fm.pad_ = 0;
    fm.lim_sum = *m.lim_acc;
    a.meta[f] = fm;
  }
}

__global__ void __launch_bounds__(kSortThreads) pnms_prep_sort_frame(PrepArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  if (frame_skipped(a.dense, blockIdx.x)) return;
  prep_sort_frame_body(a, blockIdx.x, smem_raw);
}

// the same over the binned path's declined-frame list: a small persistent grid launched
// programmatically after the binned kernel (kept separate so the full-batch kernel above keeps
// its register budget)
__global__ void __launch_bounds__(kSortThreads) pnms_prep_sort_frame_list(PrepArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  pdl_wait();
  pdl_trigger();
  const int n = *a.list_count;
  for (int li = blockIdx.x; li < n; li += gridDim.x) {
    prep_sort_frame_body(a, a.list[li], smem_raw);
    __syncthreads();
  }
}

// Chunk mode (n_max > kSortMax), grid = batch * nchunks: sort one kSortMax-slot chunk and
// publish (sorted key, input index) plus the chunk's statistics (meta is zeroed by the host).
__device__ __forceinline__ void prep_sort_chunk_body(const PrepArgs& a, int f, int c, unsigned char* smem_raw) {
  const long long fbase = (long long)f * a.n_max;
  const int cnt = frame_count(a.counts, f, a.n_max);
  const int e0 = c * kSortMax;
  // zero this chunk's share of the suppression words
  for (int w = e0 / 32 + threadIdx.x; w < min(a.W32, (e0 + kSortMax) / 32); w += kSortThreads)
    a.supp[(long long)f * a.W32 + w] = 0u;
  const int len = min(kSortMax, cnt - e0);
  if (len <= 0) return;
  SortSmem m = carve_sort_smem(smem_raw, kSortMax);
  init_stats(m.st, m.lim_acc);
  __syncthreads();
  load_keys(a, fbase, e0, len, kSortMax, m.ka, m.ia, m.st);
  __syncthreads();
  const uint32_t diff_hi = m.st->or_hi ^ m.st->and_hi;
  uint64_t* k = m.ka;
  uint16_t* id = m.ia;
  if (len > 1) block_sort_keys(&k, &id, m.kb, m.ib, m.hist, m.scan_tmp, kSortMax / kSortThreads, len, diff_hi);
  for (int p = threadIdx.x; p < len; p += kSortThreads) {
    a.sk_scratch[fbase + e0 + p] = k[p];
    a.idx_scratch[fbase + e0 + p] = e0 + id[p];
  }
  if (threadIdx.x == 0) {
    FrameMeta* fm = a.meta + f;
    atomicAdd(&fm->n_active, m.st->n_act);
    atomicMax(&fm->mode, m.st->mode);
    atomicAdd(&fm->cnt_neg, m.st->neg);
    atomicAdd(&fm->cnt_pos, m.st->pos);
    atomicAdd(&fm->cnt_zero, m.st->zero);
  }
}

__global__ void __launch_bounds__(kSortThreads) pnms_prep_sort_chunk(PrepArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  if (a.list) {
    // declined-frame list (PDL after the binned kernel; the decliner zeroed each frame's meta)
    pdl_wait();
    pdl_trigger();
    const long long n = (long long)*a.list_count * a.nchunks;
    for (long long it = blockIdx.x; it < n; it += gridDim.x) {
      prep_sort_chunk_body(a, a.list[it / a.nchunks], (int)(it % a.nchunks), smem_raw);
      __syncthreads();
    }
    return;
  }
  const int f = blockIdx.x / a.nchunks;
  if (frame_skipped(a.dense, f)) return;
  prep_sort_chunk_body(a, f, blockIdx.x % a.nchunks, smem_raw);
}

// Chunk mode, second pass: one thread per slot computes its global sorted position and its
// column limit by binary search in every chunk, then emits perm / lim / record.
__device__ __forceinline__ void merge_rank_body(const PrepArgs& a, int f, int blk) {
  const int e = blk * 256 + threadIdx.x;
  const long long fbase = (long long)f * a.n_max;
  const int cnt = frame_count(a.counts, f, a.n_max);
  unsigned long long l = 0;
  if (e < cnt) {
    const int c = e / kSortMax;
    const uint64_t* S = a.sk_scratch + fbase;
    const uint64_t sk = S[e];
    const int i = a.idx_scratch[fbase + e];
    int rank = e - c * kSortMax;
    int first = 0;
    for (int cc = 0; cc < a.nchunks; ++cc) {
      const int b = cc * kSortMax;
      const int len = min(kSortMax, cnt - b);
      if (len <= 0) break;
      const int lb = lower_bound_u64(S + b, len, sk);
      first += lb;
      if (cc < c) rank += upper_bound_u64(S + b, len, sk);
      else if (cc > c) rank += lb;
    }
    const FrameMeta fm = a.meta[f];
    if (rank < fm.n_active) l = (a.tie_break == 1) ? rank : first;
    a.perm[fbase + rank] = i;
    a.lim[fbase + rank] = (int)l;
    const long long g = fbase + i;
    write_record(a.rec + fbase * kRecBytes, rank, fm.mode, a.x[g], a.y[g], a.z[g], a.theta);
  }
  unsigned lo = __reduce_add_sync(0xFFFFFFFFu, (unsigned)(l & 0xFFFFFFFFull));
  unsigned hi = __reduce_add_sync(0xFFFFFFFFu, (unsigned)(l >> 32));
  if ((threadIdx.x & 31) == 0 && (lo | hi)) atomicAdd(&a.meta[f].lim_sum, ((unsigned long long)hi << 32) + lo);
}

__global__ void __launch_bounds__(256) pnms_merge_rank(PrepArgs a) {
  const int blocks_per_frame = (a.n_max + 255) / 256;
  if (a.list) {
    pdl_wait();
    pdl_trigger();
    const long long n = (long long)*a.list_count * blocks_per_frame;
    for (long long it = blockIdx.x; it < n; it += gridDim.x)
      merge_rank_body(a, a.list[it / blocks_per_frame], (int)(it % blocks_per_frame));
    return;
  }
  const int f = blockIdx.x / blocks_per_frame;
  if (frame_skipped(a.dense, f)) return;
  merge_rank_body(a, f, blockIdx.x % blocks_per_frame);
}

}  // namespace pnms

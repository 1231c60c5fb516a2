/*
 * parnms_b200.h — C ABI of the B200 (sm_100a) NMS engine.
 *
 * Drop-in boundary for the reference's NMS hot path
 *   engine.run_nms(d, cfg)          /root/reference/pkg/src/parnms/engine.py:296-300
 *   engine.map_phase(d, cfg)        engine.py:176-250
 *   engine.reduce_phase(b, cfg)     engine.py:253-281
 *   engine.mask_survivors(d, v)     engine.py:284-293   (host-side; uses pnms_run's keep output)
 *
 * Semantics (identical to the reference, bit for bit):
 *   row i of a frame is suppressed iff some slot j of the frame (padding included,
 *   padding = (0,0,0,0.0), detections.py:88) satisfies
 *     gate(i,j)  = s_i < s_j  or  (tie_break == by_index and s_i == s_j and i > j)   engine.py:233-235
 *     !keep(i,j) where keep = float64(w)*h < theta*(z_j+1)^2  and  z_j != 0       engine.py:219-232
 *     w = max(min(x_i+z_i, x_j+z_j) - max(x_i,x_j) + 1, 0) in int32 (same for h)
 *   survivors are the rows i < count that are not suppressed, in ascending input order
 *   (engine.py:291-292).
 *
 * Conventions: every pointer below is a DEVICE pointer unless stated otherwise; every
 * call is asynchronous on `stream` (a cudaStream_t passed as void*; NULL = legacy default
 * stream); no call allocates memory or synchronises the host.  All entry points return
 * PNMS_OK (0) or a negative pnms_status.  Asynchronous CUDA faults surface at the caller's
 * next synchronisation, exactly like any other CUDA library.
 */
#ifndef PARNMS_B200_H_
#define PARNMS_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum pnms_status {
  PNMS_OK = 0,
  PNMS_EINVAL_THETA = -1,     /* theta outside [0,1]            (engine.py:57-58 ConfigError) */
  PNMS_EINVAL_DMAX = -2,      /* d_max < 1 or count > d_max      (engine.py:59-60, 185-186)   */
  PNMS_EINVAL_TIE = -3,       /* tie_break not 0/1               (engine.py:67-71)            */
  PNMS_EINVAL_ARG = -4,       /* null pointer / negative size                                  */
  PNMS_EWORKSPACE = -5,       /* workspace missing or too small                                */
  PNMS_ETOO_LARGE = -6,       /* n_max above PNMS_MAX_SLOTS                                    */
  PNMS_ECUDA = -7,            /* a CUDA launch failed (see pnms_last_cuda_error)               */
  PNMS_EINVAL_K = -8          /* k < 1 or k does not divide d_max (engine.py:61-64)            */
} pnms_status;

/* tie_break values (NmsConfig.tie_break, engine.py:33) */
#define PNMS_TIE_PAPER_FAITHFUL 0
#define PNMS_TIE_BY_INDEX 1

/* largest per-frame slot count the batched path accepts */
#define PNMS_MAX_SLOTS 65536

/* Bytes of device workspace pnms_run needs for `batch` frames of stride `n_max`.
 * Replaces the reference's per-call SuppressionMatrix.all_ones allocation
 * (engine.py:93-96, 187).  The workspace starts with a small persistent scratch region that
 * must be zero before the first call (allocate zeroed, or call pnms_workspace_init once);
 * every call leaves it valid for the next one, so a workspace is reused across calls with no
 * clearing. */
int pnms_workspace_bytes(int batch, int n_max, size_t* out_bytes);

/* Zero the persistent scratch region of a workspace (stream-ordered). */
int pnms_workspace_init(void* workspace, size_t workspace_bytes, void* stream);

/* Batched NMS: the whole run_nms pipeline (engine.py:296-300) for `batch` frames.
 *
 *  x, y, z   int32 [batch][n_max]   box corner and side (DetectionVector._x/_y/_z cast to
 *                                   int32 as engine.py:191-193 does)
 *  s         float64 [batch][n_max] scores (DetectionVector._s)
 *  counts    int32 [batch]          valid prefix length per frame (DetectionVector.count);
 *                                   NULL means every frame has n_max valid slots.  Values are
 *                                   clamped to [0, n_max] on the device.
 *  d_max     frame capacity (NmsConfig.d_max); slots [count, d_max) are implicit PADDING
 *            (0,0,0,0.0) and take part in the gate exactly like the reference's padding
 *            columns do.  Must be >= n_max's valid counts (checked by the caller).
 *  theta     NmsConfig.theta, float64 in [0,1]
 *  tie_break PNMS_TIE_PAPER_FAITHFUL or PNMS_TIE_BY_INDEX
 * outputs (each may be NULL):
 *  keep_idx   int32 [batch][n_max]   ascending survivor indices, first keep_count[f] valid
 *  keep_count int32 [batch]          number of survivors (len(NmsResult.survivors))
 *  keep_mask  uint32 [batch][ceil(n_max/32)]  survivor bits, bit i%32 of word i/32 — the
 *             SurvivorMask of engine.py:114-131 restricted to valid rows
 *  gate_pairs uint64 [batch]         WorkCounters.map_writes of the reference's map phase
 *                                    (engine.py:236-237), padding slots included
 */
int pnms_run(const int32_t* x, const int32_t* y, const int32_t* z, const double* s,
             const int32_t* counts, int batch, int n_max, int d_max, double theta,
             int tie_break, int32_t* keep_idx, int32_t* keep_count, uint32_t* keep_mask,
             uint64_t* gate_pairs, void* workspace, size_t workspace_bytes, void* stream);

/* pnms_run plus phase timing: phase_events points at 4 cudaEvent_t handles (each may be
 * NULL) recorded on `stream` before the sort, before the map, before the compaction and
 * after it.  Used by bench.py to time the map kernel on its own launch stream. */
int pnms_run_profiled(const int32_t* x, const int32_t* y, const int32_t* z, const double* s,
                      const int32_t* counts, int batch, int n_max, int d_max, double theta, int tie_break,
                      int32_t* keep_idx, int32_t* keep_count, uint32_t* keep_mask, uint64_t* gate_pairs,
                      void* workspace, size_t workspace_bytes, void* stream, void* const* phase_events);

/* Device paths of pnms_run (every path gives the same, reference-identical result):
 *   SMALL        single launch, unsorted full pair matrix (tiny calls)
 *   BINNED       exact spatial culling, one 512-thread CTA per frame (frames <= 4096 slots)
 *   BINNED_WIDE  the same kernel with one 1024-thread CTA per SM (frames <= 2048 slots)
 *   TILES        128 independent tile CTAs per frame (latency of large single frames)
 *   CLUSTER      one thread-block cluster per frame (frames of 4097..65536 slots, batches)
 *   DENSE        sorted N x N map (prep+sort -> map -> compact), any frame
 *   COOP         one cooperative launch of up to 128 tile CTAs per frame sharing the frame's
 *                statistics and binning through global memory (latency, <= 2 frames)
 * The culling paths decline frames outside their exactness preconditions (a zero side or
 * theta = 0, coordinates outside the 15-bit domain, a crowded cell); the device finishes those
 * frames on the dense pipeline. */
#define PNMS_PATH_AUTO 0
#define PNMS_PATH_SMALL 1
#define PNMS_PATH_BINNED 2
#define PNMS_PATH_BINNED_WIDE 3
#define PNMS_PATH_TILES 4
#define PNMS_PATH_CLUSTER 5
#define PNMS_PATH_DENSE 6
#define PNMS_PATH_COOP 7

/* Launch configuration (all fields 0 = the measured defaults).  Tests, tools and the
 * benchmark use it to pin a path or a decomposition; production callers pass NULL.
 * It replaces the reference's per-call ThreadPoolExecutor shape (engine.py:156-173,
 * NmsConfig.k/workers), which never changes the result. */
typedef struct pnms_launch_config {
  int path;            /* PNMS_PATH_*; a path that cannot take the call falls back to AUTO */
  int cluster_size;    /* CLUSTER: 8 or 16 CTAs per frame (0 = 16 when co-schedulable)     */
  int cell_q8;         /* binned cells: < 0 square side -cell_q8 px, > 0 (max_z+1)*q8/256  */
  int cell_sx;         /* binned cells: > 0 overrides the cell width                       */
  int map_rows;        /* DENSE map: rows per lane 1, 2 or 4                               */
  int map_chunk;       /* DENSE map: column chunk, a multiple of 32 in [32, 4096]           */
  int small_col_tiles; /* SMALL: column tiles per frame                                    */
  int host_chain;      /* 1: the host launches the fallback chain for declined frames      */
  int32_t* declined;   /* device int32[1] or NULL: frames the culling kernel declined      */
  int binned_impl;     /* BINNED: 0 default (ranked, balanced rows), 1 first-generation     */
  int coop_tiles;      /* COOP: tile CTAs per frame (0 = one per 128 slots, 16..512)       */
} pnms_launch_config;

/* Path report of one pnms_run_ex call (host memory). */
typedef struct pnms_run_info {
  int path;            /* PNMS_PATH_* that ran (declined frames additionally ran DENSE)    */
} pnms_run_info;

/* pnms_run with an explicit launch configuration (may be NULL), a path report (may be NULL)
 * and optional phase events (as pnms_run_profiled; may be NULL). */
int pnms_run_ex(const int32_t* x, const int32_t* y, const int32_t* z, const double* s,
                const int32_t* counts, int batch, int n_max, int d_max, double theta, int tie_break,
                int32_t* keep_idx, int32_t* keep_count, uint32_t* keep_mask, uint64_t* gate_pairs,
                void* workspace, size_t workspace_bytes, void* stream, const pnms_launch_config* config,
                pnms_run_info* info, void* const* phase_events);

/* Reference-layout map phase (engine.py:176-250): writes the full d_max x d_max
 * SuppressionMatrix — row-major, rows padded to 64-bit words, bit (i,j) at word j/64 bit
 * j%64 (= byte j/8 bit j%8, little endian, engine.py:74-111), pad bits set to 1 — for ONE
 * frame whose d_max slots are all given explicitly (padding included).
 *  bits        uint64 [d_max][ceil(d_max/64)]
 *  gate_pairs  uint64 [1] (may be NULL): WorkCounters.map_writes */
int pnms_map_reference_layout(const int32_t* x, const int32_t* y, const int32_t* z,
                              const double* s, int d_max, double theta, int tie_break,
                              uint64_t* bits, uint64_t* gate_pairs, void* stream);

/* Reference reduce phase (engine.py:253-281): mask bit i = AND of the first d_max bits
 * of row i of `bits` (layout as above).  The result is independent of k (Theorem 2);
 * k is validated like NmsConfig (engine.py:61-64) and otherwise unused.
 *  mask  uint8 [ceil(d_max/8)]  packed little-endian (SurvivorMask.bits, engine.py:120-122) */
int pnms_reduce_rows(const uint64_t* bits, int d_max, int k, uint8_t* mask, void* stream);

/* Classic greedy NMS (oracles.greedy_nms, oracles.py:64-85) for `batch` frames of up to
 * PNMS_MAX_SLOTS slots: visit valid detections by (score desc, index asc), keep one unless an
 * already-kept detection covers it (positive extents on both axes and w*h >= theta*(z_ref+1)^2,
 * oracles.py:20-29).  Outputs as pnms_run (keep_idx ascending, keep_count, keep_mask; each
 * may be NULL).  Frames of up to 4096 slots need no workspace; larger frames need
 * pnms_variant_workspace_bytes() bytes (pnms_run without it returns PNMS_ETOO_LARGE for them).
 * Scores must not be NaN (the reference's ordering is undefined for NaN; here NaN detections
 * are kept and never cover others). */
int pnms_greedy_run(const int32_t* x, const int32_t* y, const int32_t* z, const double* s,
                    const int32_t* counts, int batch, int n_max, double theta, int32_t* keep_idx,
                    int32_t* keep_count, uint32_t* keep_mask, void* stream);
int pnms_greedy_run_ws(const int32_t* x, const int32_t* y, const int32_t* z, const double* s,
                       const int32_t* counts, int batch, int n_max, double theta, int32_t* keep_idx,
                       int32_t* keep_count, uint32_t* keep_mask, void* workspace, size_t workspace_bytes,
                       void* stream);

/* Device scratch the greedy and Soft-NMS kernels need for `batch` frames of stride n_max
 * (0 up to 4096 slots, where the per-slot state lives in shared memory). */
int pnms_variant_workspace_bytes(int batch, int n_max, size_t* out_bytes);

/* Soft-NMS rescoring (oracles.soft_nms_rescore, oracles.py:88-123) for `batch` frames of up
 * to PNMS_MAX_SLOTS slots (workspace as pnms_greedy_run_ws for frames over 4096 slots):
 * repeatedly select the pending detection with the highest current score
 * (ties: lowest index) and rescale every pending score by its coverage cov = w*h/(z_sel+1)^2
 * of the selected box: mode 0 (linear) s *= 1 - cov when cov >= theta; mode 1 (gaussian)
 * s *= exp(-cov^2 / sigma).  out_s [batch, n_max] float64 receives the rescored scores in
 * input order (0.0 in padding slots).  status [batch]: 0 ok, 1 a valid score is not finite
 * and > 0 (the validated domain, detections.py:79-84; frame left unwritten).  rounds
 * [batch] (may be NULL): parallel resolution rounds used.  Both modes are bit-identical to
 * the reference (gaussian: exp restated from the host libm, see pnms_debug_exp).
 * mode not 0/1 or sigma <= 0 -> PNMS_EINVAL_ARG (oracles.py:108-111). */
int pnms_soft_rescore(const int32_t* x, const int32_t* y, const int32_t* z, const double* s,
                      const int32_t* counts, int batch, int n_max, int mode, double theta, double sigma,
                      double* out_s, int32_t* status, int32_t* rounds, void* stream);
int pnms_soft_rescore_ws(const int32_t* x, const int32_t* y, const int32_t* z, const double* s,
                         const int32_t* counts, int batch, int n_max, int mode, double theta, double sigma,
                         double* out_s, int32_t* status, int32_t* rounds, void* workspace,
                         size_t workspace_bytes, void* stream);

/* Device-side ingest validation (detections.py:60-85, Detection.validate): for each frame,
 * first_bad[f] = the smallest slot index in [0, counts[f]) violating the detection invariants
 * (integer coordinates in [0, 2^24), side >= 1, finite score > 0), or -1; reason[f] says which
 * check failed (1..3 negative x/y/z, 4..6 x/y/z >= 2^24, 7 side < 1, 8 score not finite,
 * 9 score <= 0, 0 valid).  first_bad, reason: int32 [batch] device arrays. */
int pnms_validate(const int32_t* x, const int32_t* y, const int32_t* z, const double* s,
                  const int32_t* counts, int batch, int n_max, int32_t* first_bad, int32_t* reason,
                  void* stream);

/* Compact ingest: widen int16 x/y/z planes (pixel coordinates of images < 32768 px, 6 B per
 * box instead of 12) into the int32 planes pnms_run consumes.  n = number of slots. */
int pnms_widen_i16(const int16_t* x16, const int16_t* y16, const int16_t* z16, int32_t* x, int32_t* y,
                   int32_t* z, long long n, void* stream);

/* Compact ingest: unpack 32-bit boxes  box = x | y << 12 | z << 24  (x, y < 4096, z < 256:
 * frames up to 4096x4096 px, e.g. 1080p and 4K; 4 B per box instead of 12) into the int32
 * planes pnms_run consumes.  n = number of slots. */
int pnms_unpack_box32(const uint32_t* box, int32_t* x, int32_t* y, int32_t* z, long long n, void* stream);

/* Compact ingest, host side: box[i] = x[i] | y[i] << 12 | z[i] << 24 for HOST int32 planes
 * (the C ABI's own layout), on `threads` host threads (<= 0: every core), so a caller holding
 * the reference's int32 columns (engine.py:191-193) ships 4 B of geometry per box instead of 12
 * and the device unpacks them (pnms_unpack_box32).  *packable = 1 when every value is inside
 * the packable domain (x, y in [0, 4095], z in [0, 255]), else 0 — then `box` is not valid and
 * the caller sends the int32 planes.  No CUDA call; safe without a GPU. */
int pnms_pack_box32_host(const int32_t* x, const int32_t* y, const int32_t* z, long long n, uint32_t* box,
                         int threads, int* packable);

/* Diagnostics: device counter (uint64) that the binned path atomically increments by the
 * number of pair tests it executes; NULL disables (default).  Process-wide, not reentrant. */
int pnms_debug_count_pairs(uint64_t* device_counter);

/* Diagnostics: y[i] = exp(x[i]) computed on the device exactly as the host C library does
 * (pnms_libm.cuh, the exp gaussian Soft-NMS uses); x, y: float64 [n] device arrays. */
int pnms_debug_exp(const double* x, double* y, long long n, void* stream);

/* Diagnostics: device buffer of >= 256 uint64 that the large-frame kernels fill with global-timer
 * stamps (CTA r < 16, phase k < 16 at [r*16 + k]); NULL disables (default).  Process-wide. */
int pnms_debug_trace(uint64_t* device_buffer);

/* Human-readable text for a pnms_status. */
const char* pnms_strerror(int status);

/* cudaError_t of the most recent failed launch in this thread (0 if none). */
int pnms_last_cuda_error(void);

/* Library version string, e.g. "parnms_b200 0.1.0 sm_100a". */
const char* pnms_version(void);

#ifdef __cplusplus
}
#endif
#endif /* PARNMS_B200_H_ */

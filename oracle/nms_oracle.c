/*
 * nms_oracle.c — scalar C restatement of the reference engine's run_nms — TEST
 * INFRASTRUCTURE ONLY (used by tests/ and bench.py's CPU-baseline leg, never by the
 * product library).
 *
 * It follows /root/reference/pkg/src/parnms/engine.py:
 *   cell verdict     engine.py:219-239  (int32 wrap-around working copies :191-196,
 *                    float64 product vs float64 threshold :197,229-231, padding guard :232,
 *                    gate s_i < s_j (+ by_index tie clause) :233-235)
 *   row AND          engine.py:253-281  (a row survives iff no gated cell is cleared)
 *   survivor mask    engine.py:284-293  (rows < count, ascending)
 *   map_writes       engine.py:236-237  (every gate pass over the d_max x d_max slots)
 * Slots [count, d_max) are PADDING (0,0,0,0.0) as DetectionVector builds them
 * (detections.py:121-131).  It is a straight double loop with an early exit per row; it
 * shares no code with the CUDA path.
 */
#include <stdint.h>
#include <stddef.h>
#include <math.h>

typedef struct {
  int32_t x, y, z;
  double s;
} slot_t;

static slot_t slot_at(const int32_t* x, const int32_t* y, const int32_t* z, const double* s, int count, int i) {
  slot_t r;
  if (i < count) {
    r.x = x[i]; r.y = y[i]; r.z = z[i]; r.s = s[i];
  } else {
    r.x = 0; r.y = 0; r.z = 0; r.s = 0.0;
  }
  return r;
}

static int32_t wrap_add(int32_t a, int32_t b) { return (int32_t)((uint32_t)a + (uint32_t)b); }
static int32_t wrap_sub(int32_t a, int32_t b) { return (int32_t)((uint32_t)a - (uint32_t)b); }
static int32_t imin(int32_t a, int32_t b) { return a < b ? a : b; }
static int32_t imax(int32_t a, int32_t b) { return a > b ? a : b; }

/* keep bit of cell (i, j): candidate i against reference j (engine.py:219-232) */
static int cell_keep(slot_t a, slot_t b, double theta) {
  int32_t w = wrap_add(wrap_sub(imin(wrap_add(a.x, a.z), wrap_add(b.x, b.z)), imax(a.x, b.x)), 1);
  int32_t h = wrap_add(wrap_sub(imin(wrap_add(a.y, a.z), wrap_add(b.y, b.z)), imax(a.y, b.y)), 1);
  if (w < 0) w = 0;
  if (h < 0) h = 0;
  double zf = (double)b.z + 1.0;
  double thr = theta * (zf * zf);
  double prod = (double)w * (double)h;
  return (prod < thr) && (b.z != 0);
}

static int cell_gate(slot_t a, slot_t b, int i, int j, int by_index) {
  return (a.s < b.s) || (by_index && a.s == b.s && i > j);
}

/* Returns the number of survivors written to keep_out (ascending input indices). */
int oracle_run_nms(const int32_t* x, const int32_t* y, const int32_t* z, const double* s, int count, int d_max,
                   double theta, int by_index, int32_t* keep_out, unsigned long long* map_writes) {
  int kept = 0;
  for (int i = 0; i < count; ++i) {
    slot_t a = slot_at(x, y, z, s, count, i);
    int suppressed = 0;
    for (int j = 0; j < d_max && !suppressed; ++j) {
      slot_t b = slot_at(x, y, z, s, count, j);
      if (cell_gate(a, b, i, j, by_index) && !cell_keep(a, b, theta)) suppressed = 1;
    }
    if (!suppressed) keep_out[kept++] = i;
  }
  if (map_writes) {
    unsigned long long g = 0;
    for (int i = 0; i < d_max; ++i) {
      slot_t a = slot_at(x, y, z, s, count, i);
      for (int j = 0; j < d_max; ++j) g += (unsigned long long)cell_gate(a, slot_at(x, y, z, s, count, j), i, j, by_index);
    }
    *map_writes = g;
  }
  return kept;
}

/* Classic greedy NMS restated from oracles.greedy_nms (oracles.py:64-85): visit the valid
 * detections by (score desc, index asc); keep a detection unless an already-kept one covers
 * it, where covers(cand, ref) (oracles.py:20-29) needs positive extents on both axes and
 * w*h >= theta * (z_ref+1)^2 (exact integer w*h against the float64 product, as Python
 * compares int and float exactly).  Returns the number kept; keep_out ascending. */
static int greedy_covers(slot_t c, slot_t r, double theta) {
  long long w = (long long)(c.x + (long long)c.z < r.x + (long long)r.z ? c.x + (long long)c.z : r.x + (long long)r.z) -
                (long long)(c.x > r.x ? c.x : r.x) + 1;
  if (w <= 0) return 0;
  long long h = (long long)(c.y + (long long)c.z < r.y + (long long)r.z ? c.y + (long long)c.z : r.y + (long long)r.z) -
                (long long)(c.y > r.y ? c.y : r.y) + 1;
  if (h <= 0) return 0;
  long long a = ((long long)r.z + 1) * ((long long)r.z + 1);
  double thr = theta * (double)a;
  /* exact int >= float: compare against ceil(thr) in integers */
  double ct = ceil(thr);
  if (ct > 9.2e18) return 0;
  return (unsigned long long)w * (unsigned long long)h >= (unsigned long long)(long long)ct;
}

int oracle_greedy_nms(const int32_t* x, const int32_t* y, const int32_t* z, const double* s, int count,
                      double theta, int32_t* keep_out, int32_t* order_scratch, uint8_t* state_scratch) {
  /* order by (-s, i): insertion into a sorted index list (n is small in tests) */
  for (int i = 0; i < count; ++i) {
    int j = i;
    while (j > 0) {
      int o = order_scratch[j - 1];
      if (s[o] > s[i] || (s[o] == s[i] && o < i)) break;
      order_scratch[j] = o;
      --j;
    }
    order_scratch[j] = i;
  }
  for (int i = 0; i < count; ++i) state_scratch[i] = 1; /* pending */
  for (int k = 0; k < count; ++k) {
    int i = order_scratch[k];
    if (!state_scratch[i]) continue;
    state_scratch[i] = 2; /* kept */
    slot_t r = slot_at(x, y, z, s, count, i);
    for (int j = 0; j < count; ++j)
      if (state_scratch[j] == 1 && greedy_covers(slot_at(x, y, z, s, count, j), r, theta)) state_scratch[j] = 0;
  }
  int kept = 0;
  for (int i = 0; i < count; ++i)
    if (state_scratch[i] == 2) keep_out[kept++] = i;
  return kept;
}

/* Soft-NMS rescoring restated from oracles.soft_nms_rescore (oracles.py:88-123): repeatedly
 * select the pending detection with the highest current score (ties: lowest index), drop it
 * from the pending set, and rescale every pending score by the coverage of the selected box
 * (oracles.py:31-34: cov = w*h / (z_ref+1)^2 with clamped inclusive extents, computed as a
 * correctly rounded float64 quotient of exact integers, as Python's int / int is).
 *   mode 0 (linear):   if cov >= theta: s *= 1.0 - cov
 *   mode 1 (gaussian): s *= exp(-(cov * cov) / sigma)      (libm exp, as math.exp)
 * Writes the rescored scores in input order.  Quadratic per selection, like the reference. */
static double soft_coverage(slot_t c, slot_t r) {
  long long w = (long long)(c.x + (long long)c.z < r.x + (long long)r.z ? c.x + (long long)c.z : r.x + (long long)r.z) -
                (long long)(c.x > r.x ? c.x : r.x) + 1;
  long long h = (long long)(c.y + (long long)c.z < r.y + (long long)r.z ? c.y + (long long)c.z : r.y + (long long)r.z) -
                (long long)(c.y > r.y ? c.y : r.y) + 1;
  if (w < 0) w = 0;
  if (h < 0) h = 0;
  long long a = ((long long)r.z + 1) * ((long long)r.z + 1);
  return (double)(w * h) / (double)a;
}

void oracle_soft_nms(const int32_t* x, const int32_t* y, const int32_t* z, const double* s, int count, int mode,
                     double theta, double sigma, double* out_s, uint8_t* pending) {
  for (int i = 0; i < count; ++i) { out_s[i] = s[i]; pending[i] = 1; }
  for (int left = count; left > 0; --left) {
    int best = -1;
    for (int i = 0; i < count; ++i) {
      if (!pending[i]) continue;
      if (best < 0 || out_s[i] > out_s[best]) best = i;   /* min over (-s, i) */
    }
    pending[best] = 0;
    slot_t r = slot_at(x, y, z, s, count, best);
    for (int j = 0; j < count; ++j) {
      if (!pending[j]) continue;
      double cov = soft_coverage(slot_at(x, y, z, s, count, j), r);
      if (mode == 0) {
        if (cov >= theta) out_s[j] *= 1.0 - cov;
      } else {
        out_s[j] *= exp(-(cov * cov) / sigma);
      }
    }
  }
}

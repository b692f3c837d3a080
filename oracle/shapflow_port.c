/*
 * TEST INFRASTRUCTURE ONLY — a plain-C restatement of the reference hot path
 * (DistShap / shapflow, /root/reference/proj/core). It is the checker used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg; the
 * product (paper_2506_22668_b200/) never links or calls it.
 *
 * Pinned: tests/test_oracle_port.py checks every function here against the
 * compiled reference (oracle/_ref) and the golden vectors in tests/golden/
 * (SURVEY.md Appendix A plus fixtures made by tests/golden/make_golden.py).
 *
 * Each function cites the reference lines it restates.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------ Philox-4x32-10
 * philox.hpp:13-73. key = (lo, hi) of seed; counter = (lo, hi) of a running
 * block index, then (lo, hi) of the stream. A block yields two u64 draws:
 * first (b3 << 32) | b2, then (b1 << 32) | b0 (philox.hpp:21-27). */
typedef struct {
  uint32_t key[2], stream[2];
  uint64_t counter;
  uint32_t block[4];
  int have;
} port_philox;

static void philox_init(port_philox* p, uint64_t seed, uint64_t stream) {
  p->key[0] = (uint32_t)seed;
  p->key[1] = (uint32_t)(seed >> 32);
  p->stream[0] = (uint32_t)stream;
  p->stream[1] = (uint32_t)(stream >> 32);
  p->counter = 0;
  p->have = 0;
}

static void philox_refill(port_philox* p) {
  uint32_t c0 = (uint32_t)p->counter, c1 = (uint32_t)(p->counter >> 32);
  uint32_t c2 = p->stream[0], c3 = p->stream[1];
  uint32_t k0 = p->key[0], k1 = p->key[1];
  for (int r = 0; r < 10; ++r) {
    uint64_t prod0 = (uint64_t)0xD2511F53u * c0;
    uint64_t prod1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t lo0 = (uint32_t)prod0, hi0 = (uint32_t)(prod0 >> 32);
    uint32_t lo1 = (uint32_t)prod1, hi1 = (uint32_t)(prod1 >> 32);
    uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  p->block[0] = c0;
  p->block[1] = c1;
  p->block[2] = c2;
  p->block[3] = c3;
  p->counter++;
  p->have = 2;
}

static uint64_t philox_next(port_philox* p) {
  if (p->have == 0) philox_refill(p);
  --p->have;
  return ((uint64_t)p->block[2 * p->have + 1] << 32) | p->block[2 * p->have];
}

void port_philox_u64(uint64_t seed, uint64_t stream, uint64_t count,
                     uint64_t* out) {
  port_philox p;
  philox_init(&p, seed, stream);
  for (uint64_t i = 0; i < count; ++i) out[i] = philox_next(&p);
}

/* explain.cpp:37-40 */
uint64_t port_node_sampling_seed(uint64_t seed, uint32_t node) {
  return seed ^ (0x9E3779B97F4A7C15ull * ((uint64_t)node + 1));
}

/* sampler.cpp:67-77 — saturating binomial with 128-bit intermediate */
uint64_t port_binomial_or_max(uint32_t n, uint32_t s) {
  if (s > n) return 0;
  if (n - s < s) s = n - s;
  unsigned __int128 r = 1;
  for (uint32_t i = 1; i <= s; ++i) {
    r = r * (n - s + i) / i;
    if (r > (unsigned __int128)UINT64_MAX) return UINT64_MAX;
  }
  return (uint64_t)r;
}

/* ------------------------------------------------------------ size plan
 * sampler.cpp:93-151. Returns 0, or 2 on invalid input (DataError). */
typedef struct {
  double neg_rem;
  uint32_t s;
} rem_entry;

static int rem_cmp(const void* a, const void* b) {
  const rem_entry* x = (const rem_entry*)a;
  const rem_entry* y = (const rem_entry*)b;
  if (x->neg_rem < y->neg_rem) return -1;
  if (x->neg_rem > y->neg_rem) return 1;
  return (x->s > y->s) - (x->s < y->s);
}

int port_plan_sizes(uint32_t n, uint64_t k, int allow_exhaustive,
                    uint32_t* sizes, uint64_t* pairs, uint64_t* first,
                    uint64_t* nclasses, int* exhaustive, uint64_t* requested) {
  if (n < 2 || k == 0) return 2;
  if (k & 1) ++k;
  *requested = k;
  uint64_t nc = 0, next = 0;
  if (allow_exhaustive && n <= 62 && (((uint64_t)1 << n) - 2) <= k) {
    *exhaustive = 1;
    for (uint32_t s = 1; 2 * s <= n; ++s) {
      uint64_t p = port_binomial_or_max(n, s);
      if (2 * s == n) p /= 2;
      sizes[nc] = s;
      pairs[nc] = p;
      first[nc] = next;
      next += p;
      ++nc;
    }
    *nclasses = nc;
    return 0;
  }
  *exhaustive = 0;
  const uint64_t total_pairs = k / 2;
  const uint32_t half = n / 2;
  double* mass = (double*)calloc(half + 1, sizeof(double));
  uint64_t* quota = (uint64_t*)calloc(half + 1, sizeof(uint64_t));
  rem_entry* order = (rem_entry*)malloc(sizeof(rem_entry) * (half ? half : 1));
  double mass_sum = 0.0;
  for (uint32_t s = 1; s <= half; ++s) {
    double rho = (n - 1.0) / ((double)s * (double)(n - s));
    mass[s] = (2 * s == n) ? rho : 2.0 * rho;
    mass_sum += mass[s];
  }
  uint64_t assigned = 0;
  for (uint32_t s = 1; s <= half; ++s) {
    double ideal = (double)total_pairs * (mass[s] / mass_sum);
    uint64_t q = (uint64_t)floor(ideal);
    quota[s] = q;
    assigned += q;
    order[s - 1].neg_rem = -(ideal - (double)q);
    order[s - 1].s = s;
  }
  qsort(order, half, sizeof(rem_entry), rem_cmp);
  for (uint64_t i = 0; assigned < total_pairs; ++i) {
    ++quota[order[i % half].s];
    ++assigned;
  }
  for (uint32_t s = 1; s <= half; ++s) {
    if (quota[s] == 0) continue;
    sizes[nc] = s;
    pairs[nc] = quota[s];
    first[nc] = next;
    next += quota[s];
    ++nc;
  }
  *nclasses = nc;
  free(mass);
  free(quota);
  free(order);
  return 0;
}

/* ------------------------------------------------------------ masks */
static int test_bit(const uint64_t* row, uint64_t j) {
  return (int)((row[j >> 6] >> (j & 63)) & 1u);
}
static void set_bit(uint64_t* row, uint64_t j) {
  row[j >> 6] |= (uint64_t)1 << (j & 63);
}

/* sampler.cpp:38-51 */
static void unrank_combination(uint64_t* row, uint64_t idx, uint32_t m,
                               uint32_t t, uint32_t offset) {
  uint32_t x = 0;
  for (uint32_t i = 0; i < t; ++i) {
    for (;;) {
      uint64_t c = port_binomial_or_max(m - 1 - x, t - 1 - i);
      if (idx < c) break;
      idx -= c;
      ++x;
    }
    set_bit(row, x + offset);
    ++x;
  }
}

/* sampler.cpp:55-63 — Floyd with the row as its own membership set */
static void sample_subset(uint64_t* row, uint32_t n, uint32_t s,
                          port_philox* rng) {
  for (uint32_t m = n - s; m < n; ++m) {
    uint32_t t = (uint32_t)(philox_next(rng) % ((uint64_t)m + 1));
    set_bit(row, test_bit(row, t) ? m : t);
  }
}

/* sampler.cpp:153-210 for a plan given as class arrays. out receives
 * 2 * (local pairs) rows of words_for_bits(n) words; returns rows written.
 * Only global pairs g in [g_begin, g_end) with g % world == rank are
 * produced (the full shard when g_begin = 0, g_end = total pairs), so a
 * bounded slice of a large shard can be regenerated. */
uint64_t port_generate_masks(uint32_t n, const uint32_t* sizes,
                             const uint64_t* pairs, const uint64_t* first,
                             uint64_t nclasses, int exhaustive, uint64_t seed,
                             int rank, int world, uint64_t g_begin,
                             uint64_t g_end, uint64_t* out) {
  const uint64_t W = (n + 63) / 64;
  const uint64_t tail = (n % 64) ? (((uint64_t)1 << (n % 64)) - 1) : ~0ull;
  uint64_t j = 0;
  uint64_t g0 = g_begin;
  if (g0 % (uint64_t)world != (uint64_t)rank)
    g0 += ((uint64_t)rank + world - g0 % world) % world;
  uint64_t ci = 0;
  for (uint64_t g = g0; g < g_end; g += world, ++j) {
    while (ci < nclasses && g >= first[ci] + pairs[ci]) ++ci;
    uint64_t* sub = out + (2 * j) * W;
    uint64_t* comp = out + (2 * j + 1) * W;
    memset(sub, 0, W * 8);
    if (exhaustive) {
      uint64_t idx = g - first[ci];
      if (2 * sizes[ci] == n) {
        set_bit(sub, 0);
        unrank_combination(sub, idx, n - 1, sizes[ci] - 1, 1);
      } else {
        unrank_combination(sub, idx, n, sizes[ci], 0);
      }
    } else {
      port_philox rng;
      philox_init(&rng, seed, g);
      sample_subset(sub, n, sizes[ci], &rng);
    }
    for (uint64_t w = 0; w < W; ++w) comp[w] = ~sub[w];
    comp[W - 1] &= tail;
  }
  return 2 * j;
}

/* ------------------------------------------------------------ GCN forward
 * gcn.cpp:40-156 for ONE mask (every per-sample quantity is self-contained,
 * gcn.cpp:35-39, so this equals any batch size). Float arithmetic in the
 * reference order: deg counts the self-loop, isd = 1/sqrtf(deg); each row
 * aggregates self-loop first then kept neighbors in CSR order with
 * val = isd_u * isd_v; then bias-first affine; ReLU on hidden layers; the
 * last layer only at the target row (local 0); float softmax with max
 * subtraction. Writes all class probabilities into probs[C].
 *
 * dims[0..L]; weights/biases concatenated per layer (in x out row-major). */
void port_gcn_probs(uint32_t V, const uint64_t* row_ptr, const uint32_t* col,
                    const uint32_t* edge_player, const float* features,
                    int L, const uint64_t* dims, const float* weights,
                    const float* biases, const uint64_t* mask, float* probs) {
  uint64_t dmax = dims[0];
  for (int l = 1; l <= L; ++l)
    if (dims[l] > dmax) dmax = dims[l];
  float* isd = (float*)malloc(sizeof(float) * (V ? V : 1));
  float* h = (float*)malloc(sizeof(float) * (size_t)V * dmax);
  float* hn = (float*)malloc(sizeof(float) * (size_t)V * dmax);
  float* ah = (float*)malloc(sizeof(float) * (size_t)V * dmax);
  for (uint32_t u = 0; u < V; ++u) {
    uint64_t deg = 1;
    for (uint64_t i = row_ptr[u]; i < row_ptr[u + 1]; ++i)
      deg += (uint64_t)test_bit(mask, edge_player[i]);
    isd[u] = 1.0f / sqrtf((float)deg);
  }
  memcpy(h, features, sizeof(float) * (size_t)V * dims[0]);
  const float* W = weights;
  const float* B = biases;
  for (int l = 0; l < L; ++l) {
    const uint64_t din = dims[l], dout = dims[l + 1];
    const int last = (l + 1 == L);
    const uint32_t rows = last ? 1 : V;
    for (uint32_t r = 0; r < rows; ++r) {
      float* dst = ah + (size_t)r * din;
      for (uint64_t j = 0; j < din; ++j) dst[j] = 0.0f;
      { /* self-loop entry leads the row */
        const float a = isd[r] * isd[r];
        const float* src = h + (size_t)r * din;
        for (uint64_t j = 0; j < din; ++j) dst[j] += a * src[j];
      }
      for (uint64_t i = row_ptr[r]; i < row_ptr[r + 1]; ++i) {
        if (!test_bit(mask, edge_player[i])) continue;
        const float a = isd[r] * isd[col[i]];
        const float* src = h + (size_t)col[i] * din;
        for (uint64_t j = 0; j < din; ++j) dst[j] += a * src[j];
      }
    }
    for (uint32_t r = 0; r < rows; ++r) {
      const float* src = ah + (size_t)r * din;
      float* dst = last ? probs : hn + (size_t)r * dout;
      for (uint64_t j = 0; j < dout; ++j) dst[j] = B[j];
      for (uint64_t kin = 0; kin < din; ++kin) {
        const float a = src[kin];
        const float* wrow = W + kin * dout;
        for (uint64_t j = 0; j < dout; ++j) dst[j] += a * wrow[j];
      }
      if (!last)
        for (uint64_t j = 0; j < dout; ++j) dst[j] = dst[j] > 0.0f ? dst[j] : 0.0f;
    }
    if (!last) {
      float* t = h;
      h = hn;
      hn = t;
    }
    W += din * dout;
    B += dout;
  }
  const uint64_t C = dims[L];
  float mx = probs[0];
  for (uint64_t c = 1; c < C; ++c) mx = probs[c] > mx ? probs[c] : mx;
  float sum = 0.0f;
  for (uint64_t c = 0; c < C; ++c) {
    probs[c] = expf(probs[c] - mx);
    sum += probs[c];
  }
  for (uint64_t c = 0; c < C; ++c) probs[c] /= sum;
  free(isd);
  free(h);
  free(hn);
  free(ah);
}

/* predict_batched (gcn.cpp:259-270): p[class] per mask row */
void port_gcn_predict(uint32_t V, const uint64_t* row_ptr, const uint32_t* col,
                      const uint32_t* edge_player, const float* features,
                      int L, const uint64_t* dims, const float* weights,
                      const float* biases, const uint64_t* bits, uint64_t rows,
                      uint64_t words, uint32_t cls, float* out) {
  float* probs = (float*)malloc(sizeof(float) * dims[L]);
  for (uint64_t r = 0; r < rows; ++r) {
    port_gcn_probs(V, row_ptr, col, edge_player, features, L, dims, weights,
                   biases, bits + r * words, probs);
    out[r] = probs[cls];
  }
  free(probs);
}

/* ------------------------------------------------------------ CGLS on bit rows
 * assemble_problem (solver.cpp:95-156) + solve_cgls (solver.cpp:158-362),
 * one worker, restated over bit rows instead of dense float rows. The dense
 * reference adds 0.0 * u[i] (or co + beta * 0.0) for clear bits; the dot
 * products here skip those terms and the transpose leaves write co exactly,
 * which leaves every sum bitwise unchanged (adding +0.0 to a finite sum is
 * the identity, and beta * 0.0 = +-0.0). Fixed-order folding follows the
 * PairwiseFolder (solver.cpp:31-61) with bit-reversed leaves (228-237).
 *
 * rows_of_size: n+1 global per-size row counts (sampler.cpp:168-176).
 * Returns 0, 2 (DataError) or 3 (NumericalError). */
static uint64_t bit_ceil64(uint64_t x) {
  uint64_t r = 1;
  while (r < x) r <<= 1;
  return r;
}

static uint64_t bit_reverse(uint64_t x, int bits) {
  uint64_t r = 0;
  for (int b = 0; b < bits; ++b) {
    r = (r << 1) | (x & 1);
    x >>= 1;
  }
  return r;
}

typedef struct {
  size_t len;
  uint64_t count;
  double* carry;
  double** slots;
  int nslots;
} folder;

static void folder_init(folder* f, size_t len) {
  f->len = len;
  f->count = 0;
  f->carry = (double*)calloc(len ? len : 1, sizeof(double));
  f->slots = (double**)calloc(64, sizeof(double*));
  f->nslots = 0;
}
static void folder_free(folder* f) {
  free(f->carry);
  for (int i = 0; i < 64; ++i) free(f->slots[i]);
  free(f->slots);
}
static void folder_push(folder* f, const double* leaf) {
  memcpy(f->carry, leaf, f->len * sizeof(double));
  int level = 0;
  for (uint64_t c = f->count; c & 1; c >>= 1, ++level) {
    const double* slot = f->slots[level];
    for (size_t i = 0; i < f->len; ++i) f->carry[i] = slot[i] + f->carry[i];
  }
  if (!f->slots[level]) f->slots[level] = (double*)calloc(f->len ? f->len : 1, sizeof(double));
  double* t = f->slots[level];
  f->slots[level] = f->carry;
  f->carry = t;
  f->count++;
}
static void folder_result(const folder* f, double* out) {
  int top = 0;
  while (!((f->count >> top) & 1)) ++top;
  memcpy(out, f->slots[top], f->len * sizeof(double));
}

int port_cgls(uint32_t n, const uint64_t* bits, uint64_t rows, uint64_t words,
              const uint64_t* rows_of_size, uint64_t global_pair_count,
              const double* values, double base, double full, double cscale,
              double tol, uint64_t max_iter, int fixed_order, double* phi,
              uint64_t* iters_out, double* resid_out, int* converged_out) {
  *iters_out = 0;
  *resid_out = 0.0;
  *converged_out = 0;
  if (n == 0) {
    *converged_out = 1;
    return 0;
  }
  if (rows % 2) return 2;
  /* weight per size (solver.cpp:125-138) */
  double* wsize = (double*)calloc(n + 1, sizeof(double));
  double scale = 0.0;
  for (uint32_t s = 1; s < n; ++s) {
    if (rows_of_size[s] == 0) continue;
    const double rho = (n - 1.0) / ((double)s * (double)(n - s));
    const double w = rho / (double)rows_of_size[s];
    if (scale == 0.0) scale = w;
    wsize[s] = w / scale;
  }
  const uint64_t pl = rows / 2;
  uint64_t pg = global_pair_count < 64 ? 64 : global_pair_count;
  pg = bit_ceil64(pg);
  uint64_t plocal = pg;
  if (pl > plocal) plocal = pl;
  plocal = bit_ceil64(plocal);
  int log_local = 0;
  while (((uint64_t)1 << log_local) < plocal) ++log_local;

  double* sw = (double*)malloc(sizeof(double) * rows);
  double* r = (double*)malloc(sizeof(double) * rows);
  double* v = (double*)malloc(sizeof(double) * rows);
  uint8_t* is_comp = (uint8_t*)malloc(pl ? pl : 1);
  int rc = 0;
  const uint64_t tail = (n % 64) ? (((uint64_t)1 << (n % 64)) - 1) : ~0ull;
  for (uint64_t i = 0; i < rows; ++i) {
    uint64_t size = 0;
    for (uint64_t w = 0; w < words; ++w) size += (uint64_t)__builtin_popcountll(bits[i * words + w]);
    if (size == 0 || size >= n) rc = 2;
    sw[i] = sqrt(wsize[size < n ? size : 0]);
    r[i] = sw[i] * (values[i] - base);
  }
  for (uint64_t j = 0; j < pl; ++j) {
    const uint64_t* e = bits + 2 * j * words;
    const uint64_t* o = e + words;
    is_comp[j] = 1;
    for (uint64_t w = 0; w < words; ++w) {
      uint64_t want = ~e[w];
      if (w == words - 1) want &= tail;
      if (o[w] != want) is_comp[j] = 0;
    }
  }
  const double sc = sqrt(cscale);
  double r_c = sc * (full - base);
  double* s = (double*)calloc(n, sizeof(double));
  double* u = (double*)calloc(n, sizeof(double));
  double* leaf = (double*)calloc(n, sizeof(double));
  folder vf, sf;
  folder_init(&vf, n);
  folder_init(&sf, 1);
  memset(phi, 0, sizeof(double) * n);
  if (rc) goto done;

#define TRANSPOSE_LEAF(J)                                                  \
  do {                                                                     \
    const uint64_t e_ = 2 * (J);                                           \
    const double ce = sw[e_] * r[e_], co = sw[e_ + 1] * r[e_ + 1];         \
    const uint64_t* re = bits + e_ * words;                                \
    if (is_comp[J]) {                                                      \
      const double beta = ce - co;                                         \
      for (uint32_t i = 0; i < n; ++i)                                     \
        leaf[i] = test_bit(re, i) ? co + beta * 1.0 : co + beta * 0.0;     \
    } else {                                                               \
      const uint64_t* ro = re + words;                                     \
      for (uint32_t i = 0; i < n; ++i)                                     \
        leaf[i] = ce * (double)test_bit(re, i) + co * (double)test_bit(ro, i); \
    }                                                                      \
  } while (0)

#define TRANSPOSE_PRODUCT()                                                \
  do {                                                                     \
    if (fixed_order) {                                                     \
      vf.count = 0;                                                        \
      for (uint64_t t = 0; t < plocal; ++t) {                              \
        const uint64_t j = bit_reverse(t, log_local);                      \
        if (j < pl)                                                        \
          TRANSPOSE_LEAF(j);                                               \
        else                                                               \
          memset(leaf, 0, sizeof(double) * n);                             \
        folder_push(&vf, leaf);                                            \
      }                                                                    \
      folder_result(&vf, s);                                               \
    } else {                                                               \
      memset(s, 0, sizeof(double) * n);                                    \
      for (uint64_t j = 0; j < pl; ++j) {                                  \
        TRANSPOSE_LEAF(j);                                                 \
        for (uint32_t i = 0; i < n; ++i) s[i] += leaf[i];                  \
      }                                                                    \
    }                                                                      \
    const double pin = sc * r_c;                                           \
    for (uint32_t i = 0; i < n; ++i) s[i] += pin;                          \
  } while (0)

  TRANSPOSE_PRODUCT();
  double gamma = 0.0;
  for (uint32_t i = 0; i < n; ++i) gamma += s[i] * s[i];
  const double gamma0 = gamma;
  if (gamma0 == 0.0) {
    *converged_out = 1;
    goto done;
  }
  double data0 = 0.0;
  {
    const double pin = sc * r_c;
    for (uint32_t i = 0; i < n; ++i) {
      const double d = s[i] - pin;
      data0 += d * d;
    }
  }
  const double reference = data0 > 0.0 ? data0 : gamma0;
  double rel = sqrt(gamma0 / reference);
  memcpy(u, s, sizeof(double) * n);
  const double blowup = 1.0e12 * (rel > 1.0 ? rel : 1.0);
  const uint64_t maxit = max_iter ? max_iter : (n < 5000 ? n : 5000);
  uint64_t it = 0;
  int conv = 0;
  while (it < maxit) {
    double sum_u = 0.0;
    for (uint32_t i = 0; i < n; ++i) sum_u += u[i];
    for (uint64_t j = 0; j < pl; ++j) {
      const uint64_t e = 2 * j;
      const uint64_t* re = bits + e * words;
      double dot = 0.0;
      for (uint32_t i = 0; i < n; ++i)
        if (test_bit(re, i)) dot += u[i];
      v[e] = sw[e] * dot;
      if (is_comp[j]) {
        v[e + 1] = sw[e + 1] * (sum_u - dot);
      } else {
        const uint64_t* ro = re + words;
        double d2 = 0.0;
        for (uint32_t i = 0; i < n; ++i)
          if (test_bit(ro, i)) d2 += u[i];
        v[e + 1] = sw[e + 1] * d2;
      }
    }
    double delta = 0.0;
    if (fixed_order) {
      sf.count = 0;
      for (uint64_t t = 0; t < plocal; ++t) {
        const uint64_t j = bit_reverse(t, log_local);
        double d = 0.0;
        if (j < pl) d = v[2 * j] * v[2 * j] + v[2 * j + 1] * v[2 * j + 1];
        folder_push(&sf, &d);
      }
      folder_result(&sf, &delta);
    } else {
      for (uint64_t i = 0; i < rows; ++i) delta += v[i] * v[i];
    }
    const double v_c = sc * sum_u;
    delta += v_c * v_c;
    if (!isfinite(delta)) {
      rc = 3;
      break;
    }
    if (delta <= 0.0) break;
    const double theta = gamma / delta;
    for (uint32_t i = 0; i < n; ++i) phi[i] += theta * u[i];
    for (uint64_t i = 0; i < rows; ++i) r[i] -= theta * v[i];
    r_c -= theta * v_c;
    TRANSPOSE_PRODUCT();
    double gn = 0.0;
    for (uint32_t i = 0; i < n; ++i) gn += s[i] * s[i];
    ++it;
    rel = sqrt(gn / reference);
    if (!isfinite(gn) || rel > blowup) {
      rc = 3;
      break;
    }
    if (rel <= tol) {
      conv = 1;
      break;
    }
    const double beta = gn / gamma;
    for (uint32_t i = 0; i < n; ++i) u[i] = s[i] + beta * u[i];
    gamma = gn;
  }
  *iters_out = it;
  *resid_out = rel;
  *converged_out = conv;
#undef TRANSPOSE_LEAF
#undef TRANSPOSE_PRODUCT
done:
  folder_free(&vf);
  folder_free(&sf);
  free(wsize);
  free(sw);
  free(r);
  free(v);
  free(is_comp);
  free(s);
  free(u);
  free(leaf);
  return rc;
}

/* solver.cpp:430-440 — descending phi, ties to the smaller index */
static const double* g_rank_phi;
static int rank_cmp(const void* a, const void* b) {
  uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  double px = g_rank_phi[x], py = g_rank_phi[y];
  if (px != py) return px > py ? -1 : 1;
  return (x > y) - (x < y);
}
void port_rank_edges(const double* phi, uint32_t n, uint32_t* order) {
  for (uint32_t i = 0; i < n; ++i) order[i] = i;
  g_rank_phi = phi;
  qsort(order, n, sizeof(uint32_t), rank_cmp);
}

/* ------------------------------------------------------------ CGLS, large k·n
 * The same algorithm as port_cgls (solver.cpp:158-362: assemble weights
 * 125-138, targets 153, pin row 111-112, complement fast paths 209-223 and
 * 261-263, stop rule / blow-up / non-finite checks 289-360) for shapes where
 * the dense leaves of the fixed-order tree are infeasible (C2: 250K pairs x
 * 50K players). Differences from port_cgls, all inside the 1e-3 parity bar:
 *   - sums over pairs run in per-thread blocks folded in thread order (not the
 *     PairwiseFolder tree), so results agree with port_cgls / the reference to
 *     rounding (tests/test_oracle_port.py pins this at ~1e-12);
 *   - M^T r visits only the set bits of each pair's even row:
 *     s_i = sum_j co_j + sum_{j : bit_e(i)} (ce_j - co_j) for complement pairs
 *     (the reference's leaf co + beta * bit, solver.cpp:209-217).
 * `threads` worker threads (pthreads); rows of size 0 or n are a DataError. */
#include <pthread.h>

typedef struct {
  uint32_t n;
  const uint64_t* bits;
  uint64_t words, pl, j0, j1;
  const double* sw;
  const double* r;
  double* v;
  const uint8_t* is_comp;
  const double* u;
  double sum_u;
  double* s_part; /* n doubles: this thread's transpose partial */
  double acc;     /* this thread's scalar partial */
  int op;         /* 0 forward, 1 transpose */
} cg_task;

static void* cg_worker(void* arg) {
  cg_task* t = (cg_task*)arg;
  const uint64_t W = t->words;
  if (t->op == 0) {
    double acc = 0.0;
    for (uint64_t j = t->j0; j < t->j1; ++j) {
      const uint64_t e = 2 * j;
      const uint64_t* re = t->bits + e * W;
      double dot = 0.0;
      for (uint64_t w = 0; w < W; ++w)
        for (uint64_t x = re[w]; x; x &= x - 1) dot += t->u[w * 64 + (uint64_t)__builtin_ctzll(x)];
      t->v[e] = t->sw[e] * dot;
      if (t->is_comp[j]) {
        t->v[e + 1] = t->sw[e + 1] * (t->sum_u - dot);
      } else {
        const uint64_t* ro = re + W;
        double d2 = 0.0;
        for (uint64_t w = 0; w < W; ++w)
          for (uint64_t x = ro[w]; x; x &= x - 1) d2 += t->u[w * 64 + (uint64_t)__builtin_ctzll(x)];
        t->v[e + 1] = t->sw[e + 1] * d2;
      }
      acc += t->v[e] * t->v[e] + t->v[e + 1] * t->v[e + 1];
    }
    t->acc = acc;
  } else {
    double* s = t->s_part;
    memset(s, 0, sizeof(double) * t->n);
    double cbase = 0.0;
    for (uint64_t j = t->j0; j < t->j1; ++j) {
      const uint64_t e = 2 * j;
      const double ce = t->sw[e] * t->r[e], co = t->sw[e + 1] * t->r[e + 1];
      const uint64_t* re = t->bits + e * W;
      if (t->is_comp[j]) {
        cbase += co;
        const double beta = ce - co;
        for (uint64_t w = 0; w < W; ++w)
          for (uint64_t x = re[w]; x; x &= x - 1) s[w * 64 + (uint64_t)__builtin_ctzll(x)] += beta;
      } else {
        const uint64_t* ro = re + W;
        for (uint64_t w = 0; w < W; ++w) {
          for (uint64_t x = re[w]; x; x &= x - 1) s[w * 64 + (uint64_t)__builtin_ctzll(x)] += ce;
          for (uint64_t x = ro[w]; x; x &= x - 1) s[w * 64 + (uint64_t)__builtin_ctzll(x)] += co;
        }
      }
    }
    t->acc = cbase;
  }
  return NULL;
}

static void cg_run(cg_task* tasks, int threads) {
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  for (int i = 1; i < threads; ++i) pthread_create(&th[i], NULL, cg_worker, &tasks[i]);
  cg_worker(&tasks[0]);
  for (int i = 1; i < threads; ++i) pthread_join(th[i], NULL);
  free(th);
}

int port_cgls_sparse(uint32_t n, const uint64_t* bits, uint64_t rows, uint64_t words,
                     const uint64_t* rows_of_size, const double* values, double base, double full,
                     double cscale, double tol, uint64_t max_iter, int threads, double* phi,
                     uint64_t* iters_out, double* resid_out, int* converged_out) {
  *iters_out = 0;
  *resid_out = 0.0;
  *converged_out = 0;
  memset(phi, 0, sizeof(double) * n);
  if (n == 0) {
    *converged_out = 1;
    return 0;
  }
  if (rows % 2) return 2;
  if (threads < 1) threads = 1;
  double* wsize = (double*)calloc(n + 1, sizeof(double));
  double scale = 0.0;
  for (uint32_t sz = 1; sz < n; ++sz) {
    if (rows_of_size[sz] == 0) continue;
    const double rho = (n - 1.0) / ((double)sz * (double)(n - sz));
    const double w = rho / (double)rows_of_size[sz];
    if (scale == 0.0) scale = w;
    wsize[sz] = w / scale;
  }
  const uint64_t pl = rows / 2;
  double* sw = (double*)malloc(sizeof(double) * (rows ? rows : 1));
  double* r = (double*)malloc(sizeof(double) * (rows ? rows : 1));
  double* v = (double*)malloc(sizeof(double) * (rows ? rows : 1));
  uint8_t* is_comp = (uint8_t*)malloc(pl ? pl : 1);
  double* s = (double*)calloc(n, sizeof(double));
  double* u = (double*)calloc(n, sizeof(double));
  double* parts = (double*)malloc(sizeof(double) * (size_t)n * (size_t)threads);
  cg_task* tasks = (cg_task*)calloc((size_t)threads, sizeof(cg_task));
  int rc = 0;
  const uint64_t tail = (n % 64) ? (((uint64_t)1 << (n % 64)) - 1) : ~0ull;
  for (uint64_t i = 0; i < rows; ++i) {
    uint64_t size = 0;
    for (uint64_t w = 0; w < words; ++w) size += (uint64_t)__builtin_popcountll(bits[i * words + w]);
    if (size == 0 || size >= n) rc = 2;
    sw[i] = sqrt(wsize[size < n ? size : 0]);
    r[i] = sw[i] * (values[i] - base);
  }
  for (uint64_t j = 0; j < pl; ++j) {
    const uint64_t* e = bits + 2 * j * words;
    const uint64_t* o = e + words;
    is_comp[j] = 1;
    for (uint64_t w = 0; w < words; ++w) {
      uint64_t want = ~e[w];
      if (w == words - 1) want &= tail;
      if (o[w] != want) is_comp[j] = 0;
    }
  }
  for (int t = 0; t < threads; ++t) {
    tasks[t].n = n;
    tasks[t].bits = bits;
    tasks[t].words = words;
    tasks[t].pl = pl;
    tasks[t].j0 = pl * (uint64_t)t / (uint64_t)threads;
    tasks[t].j1 = pl * (uint64_t)(t + 1) / (uint64_t)threads;
    tasks[t].sw = sw;
    tasks[t].r = r;
    tasks[t].v = v;
    tasks[t].is_comp = is_comp;
    tasks[t].u = u;
    tasks[t].s_part = parts + (size_t)n * (size_t)t;
  }
  const double sc = sqrt(cscale);
  double r_c = sc * (full - base);
  if (rc) goto done;

#define SPARSE_TRANSPOSE()                                                 \
  do {                                                                     \
    for (int t_ = 0; t_ < threads; ++t_) tasks[t_].op = 1;                 \
    cg_run(tasks, threads);                                                \
    double cb_ = 0.0;                                                      \
    for (int t_ = 0; t_ < threads; ++t_) cb_ += tasks[t_].acc;             \
    const double pin_ = sc * r_c;                                          \
    for (uint32_t i = 0; i < n; ++i) {                                     \
      double x_ = 0.0;                                                     \
      for (int t_ = 0; t_ < threads; ++t_) x_ += parts[(size_t)n * t_ + i]; \
      s[i] = (cb_ + x_) + pin_;                                            \
    }                                                                      \
  } while (0)

  SPARSE_TRANSPOSE();
  double gamma = 0.0;
  for (uint32_t i = 0; i < n; ++i) gamma += s[i] * s[i];
  const double gamma0 = gamma;
  if (gamma0 == 0.0) {
    *converged_out = 1;
    goto done;
  }
  double data0 = 0.0;
  {
    const double pin = sc * r_c;
    for (uint32_t i = 0; i < n; ++i) {
      const double d = s[i] - pin;
      data0 += d * d;
    }
  }
  const double reference = data0 > 0.0 ? data0 : gamma0;
  double rel = sqrt(gamma0 / reference);
  memcpy(u, s, sizeof(double) * n);
  const double blowup = 1.0e12 * (rel > 1.0 ? rel : 1.0);
  const uint64_t maxit = max_iter ? max_iter : (n < 5000 ? n : 5000);
  uint64_t it = 0;
  int conv = 0;
  while (it < maxit) {
    double sum_u = 0.0;
    for (uint32_t i = 0; i < n; ++i) sum_u += u[i];
    for (int t = 0; t < threads; ++t) {
      tasks[t].op = 0;
      tasks[t].sum_u = sum_u;
    }
    cg_run(tasks, threads);
    double delta = 0.0;
    for (int t = 0; t < threads; ++t) delta += tasks[t].acc;
    const double v_c = sc * sum_u;
    delta += v_c * v_c;
    if (!isfinite(delta)) {
      rc = 3;
      break;
    }
    if (delta <= 0.0) break;
    const double theta = gamma / delta;
    for (uint32_t i = 0; i < n; ++i) phi[i] += theta * u[i];
    for (uint64_t i = 0; i < rows; ++i) r[i] -= theta * v[i];
    r_c -= theta * v_c;
    SPARSE_TRANSPOSE();
    double gn = 0.0;
    for (uint32_t i = 0; i < n; ++i) gn += s[i] * s[i];
    ++it;
    rel = sqrt(gn / reference);
    if (!isfinite(gn) || rel > blowup) {
      rc = 3;
      break;
    }
    if (rel <= tol) {
      conv = 1;
      break;
    }
    const double beta = gn / gamma;
    for (uint32_t i = 0; i < n; ++i) u[i] = s[i] + beta * u[i];
    gamma = gn;
  }
  *iters_out = it;
  *resid_out = rel;
  *converged_out = conv;
#undef SPARSE_TRANSPOSE
done:
  free(wsize);
  free(sw);
  free(r);
  free(v);
  free(is_comp);
  free(s);
  free(u);
  free(parts);
  free(tasks);
  return rc;
}

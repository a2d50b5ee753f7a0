// Device utilities shared by the ctcb kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define CTCB_LN2 0.693147180559945309417232121458176568

namespace ctcb {

constexpr unsigned FULL = 0xffffffffu;

// ---------------------------------------------------------------- ordering
// Order-preserving unsigned key of an fp32 value (float comparison semantics:
// -0.0 and +0.0 map to the same key, as numpy's lexsort compares them equal).
__device__ __forceinline__ uint32_t ord32(float x) {
  uint32_t u = __float_as_uint(__fadd_rn(x, 0.0f));
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float unord32(uint32_t k) {
  uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(u);
}
// Order-preserving key of an fp64 score.
__device__ __forceinline__ uint64_t ord64(double d) {
  if (d == 0.0) d = 0.0;
  uint64_t u = (uint64_t)__double_as_longlong(d);
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}

// log1p(exp(-d)) for d >= 0 in ~45 branch-free fp64 instructions (CUDA's
// exp + log1p expand to ~280 inline instructions each call site).  Absolute
// error <= 2.3e-16 over d in [0, 700) (validated against numpy on 2.1M points,
// see DESIGN.md §2); the result is added to a score, so it rounds like
// numpy's log1p(exp(.)) up to one ulp of the score.
__device__ __forceinline__ double log1pexp_neg(double d) {
  const double kLog2e = 1.4426950408889634, kLn2Hi = 0.6931471803691238, kLn2Lo = 1.9082149292705877e-10;
  // exp(-d) = 2^n * exp(g), n = rint(-d*log2e), |g| <= ln2/2 (Cody-Waite)
  const double n = rint(-d * kLog2e);
  const double g = fma(-n, kLn2Lo, fma(-n, kLn2Hi, -d));
#ifdef CTCB_LAE_HORNER
  double p = 1.0 / 6227020800.0;  // 1/13!
  p = fma(p, g, 1.0 / 479001600.0);
  p = fma(p, g, 1.0 / 39916800.0);
  p = fma(p, g, 1.0 / 3628800.0);
  p = fma(p, g, 1.0 / 362880.0);
  p = fma(p, g, 1.0 / 40320.0);
  p = fma(p, g, 1.0 / 5040.0);
  p = fma(p, g, 1.0 / 720.0);
  p = fma(p, g, 1.0 / 120.0);
  p = fma(p, g, 1.0 / 24.0);
  p = fma(p, g, 1.0 / 6.0);
  p = fma(p, g, 0.5);
  p = fma(p, g, 1.0);
  p = fma(p, g, 1.0);
#else
  // Estrin evaluation of sum_{i<=13} g^i / i!: the frame step is bound by
  // dependent-latency chains, so a 5-deep tree beats the 13-deep Horner chain
  const double g2 = g * g, g4 = g2 * g2, g8 = g4 * g4;
  const double c01 = fma(g, 1.0, 1.0), c23 = fma(g, 1.0 / 6.0, 0.5);
  const double c45 = fma(g, 1.0 / 120.0, 1.0 / 24.0), c67 = fma(g, 1.0 / 5040.0, 1.0 / 720.0);
  const double c89 = fma(g, 1.0 / 362880.0, 1.0 / 40320.0), cab = fma(g, 1.0 / 39916800.0, 1.0 / 3628800.0);
  const double ccd = fma(g, 1.0 / 6227020800.0, 1.0 / 479001600.0);
  const double d03 = fma(g2, c23, c01), d47 = fma(g2, c67, c45), d8b = fma(g2, cab, c89);
  const double e07 = fma(g4, d47, d03), e8f = fma(g4, ccd, d8b);
  const double p = fma(g8, e8f, e07);
#endif
  const int ni = d < 700.0 ? (int)n : -1100;
  const double e = ni > -1022 ? p * __longlong_as_double((long long)(ni + 1023) << 52) : 0.0;
  // log1p(e) = log(z), z = 1 + e in (1, 2]: split at sqrt(2), atanh series
  const double z = 1.0 + e;
  const bool big = z > 1.4142135623730951;
  const double zz = big ? 0.5 * z : z;
  const double corr = big ? 0.5 * (e - (z - 1.0)) : (e - (z - 1.0));  // rounding of 1 + e
  const double num = zz - 1.0, den = zz + 1.0;
  double r = (double)__frcp_rn((float)den);  // 1/den: fp32 seed + two Newton steps
  r = fma(r, fma(-den, r, 1.0), r);
  r = fma(r, fma(-den, r, 1.0), r);
  double u = num * r;
  u = fma(r, fma(-den, u, num), u);
  const double u2 = u * u;
#ifdef CTCB_LAE_HORNER
  double s = 1.0 / 23.0;
  s = fma(s, u2, 1.0 / 21.0);
  s = fma(s, u2, 1.0 / 19.0);
  s = fma(s, u2, 1.0 / 17.0);
  s = fma(s, u2, 1.0 / 15.0);
  s = fma(s, u2, 1.0 / 13.0);
  s = fma(s, u2, 1.0 / 11.0);
  s = fma(s, u2, 1.0 / 9.0);
  s = fma(s, u2, 1.0 / 7.0);
  s = fma(s, u2, 1.0 / 5.0);
  s = fma(s, u2, 1.0 / 3.0);
#else
  // sum_{i=0..10} u2^i / (2i+3), Estrin
  const double w2 = u2 * u2, w4 = w2 * w2, w8 = w4 * w4;
  const double a01 = fma(u2, 1.0 / 5.0, 1.0 / 3.0), a23 = fma(u2, 1.0 / 9.0, 1.0 / 7.0);
  const double a45 = fma(u2, 1.0 / 13.0, 1.0 / 11.0), a67 = fma(u2, 1.0 / 17.0, 1.0 / 15.0);
  const double a89 = fma(u2, 1.0 / 21.0, 1.0 / 19.0);
  const double b03 = fma(w2, a23, a01), b47 = fma(w2, a67, a45), b8a = fma(w2, 1.0 / 23.0, a89);
  const double s = fma(w8, b8a, fma(w4, b47, b03));
#endif
  double res = fma(2.0 * u, u2 * s, 2.0 * u) + corr * (double)__frcp_rn((float)zz);
  return big ? res + kLn2Hi + kLn2Lo : res;
}

// log1p(exp(-d)) the way numpy's logaddexp composes it from libm: exp(-d)
// rounded to double, then log1p of that double rounded to double.  Each step
// is evaluated in double-double (~1e-29 relative) and rounded once (correct
// rounding).  glibc's log1p is not always correctly rounded, so this matches
// numpy's logaddexp on 99.74 % of random score pairs against 99.12 % for the
// polynomial (tools/micro/lae_check.py, 4 M pairs).  ~10x the instructions of
// log1pexp_neg: it only runs behind the guard in add_log1pexp_exact, and only
// the generic kernel (large beams, where quantized inputs make exact score
// ties common) uses it; the fast and fused kernels keep the polynomial.
struct ddv { double hi, lo; };
__device__ __forceinline__ ddv dd_two_sum(double a, double b) {
  const double s = __dadd_rn(a, b), bb = __dsub_rn(s, a);
  return {s, __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb))};
}
__device__ __forceinline__ ddv dd_quick(double a, double b) {
  const double s = __dadd_rn(a, b);
  return {s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ ddv dd_add(ddv a, ddv b) {
  ddv s = dd_two_sum(a.hi, b.hi);
  const ddv t = dd_two_sum(a.lo, b.lo);
  s = dd_quick(s.hi, __dadd_rn(s.lo, t.hi));
  return dd_quick(s.hi, __dadd_rn(s.lo, t.lo));
}
__device__ __forceinline__ ddv dd_mul(ddv a, ddv b) {
  const double p = __dmul_rn(a.hi, b.hi);
  const double e = fma(a.hi, b.hi, -p);
  return dd_quick(p, fma(a.hi, b.lo, fma(a.lo, b.hi, e)));
}
// exp(y) for y in [-745, 0] in double-double: y = n ln2 + r (three-part ln2),
// Taylor to degree 9 on r / 2^10, ten squarings, scale by 2^n
__device__ __forceinline__ ddv dd_exp(ddv y) {
  const double kH = 0.6931471805599453, kM = 2.3190468138462996e-17, kL = 5.707708438416212e-34;
  const double n = rint(y.hi * 1.4426950408889634);
  const double p = __dmul_rn(n, kH), pe = fma(n, kH, -p);
  ddv r = dd_add(y, {-p, -pe});
  const double q = __dmul_rn(n, kM), qe = fma(n, kM, -q);
  r = dd_add(r, {-q, -qe});
  r = dd_add(r, {-n * kL, 0.0});
  r.hi = ldexp(r.hi, -10);
  r.lo = ldexp(r.lo, -10);
  ddv s = {1.0 / 362880.0, 0.0};
  s = dd_add(dd_mul(s, r), {1.0 / 40320.0, 0.0});
  s = dd_add(dd_mul(s, r), {1.0 / 5040.0, 0.0});
  s = dd_add(dd_mul(s, r), {0.001388888888888889, -5.300543954373577e-20});   // 1/720
  s = dd_add(dd_mul(s, r), {0.008333333333333333, 1.1564823173178714e-19});   // 1/120
  s = dd_add(dd_mul(s, r), {0.041666666666666664, 2.3129646346357427e-18});   // 1/24
  s = dd_add(dd_mul(s, r), {0.16666666666666666, 9.25185853854297e-18});      // 1/6
  s = dd_add(dd_mul(s, r), {0.5, 0.0});
  s = dd_add(dd_mul(s, r), {1.0, 0.0});
  s = dd_add(dd_mul(s, r), {1.0, 0.0});
#pragma unroll
  for (int i = 0; i < 10; i++) s = dd_mul(s, s);
  const int ni = (int)n;
  return {ldexp(s.hi, ni), ldexp(s.lo, ni)};
}
__device__ __forceinline__ double log1pexp_cr(double d) {
  if (!(d < 745.0)) return 0.0;            // exp(-d) underflows to 0
  const double e = dd_exp({-d, 0.0}).hi;  // exp(-d), rounded
  const ddv z = dd_two_sum(1.0, e);        // 1 + e, exact
  const double y0 = log(z.hi);
  const ddv w = dd_mul(z, dd_exp({-y0, 0.0}));
  return dd_add({y0, 0.0}, dd_add(w, {-1.0, 0.0})).hi;  // one Newton step for log(1 + e)
}

// big + log1p(exp(-d)): the polynomial first; when the sum is within the
// polynomial's error (+ half an ulp of the term) of a rounding boundary of
// `big + term`, recompute the term with log1pexp_cr.
__device__ __forceinline__ double add_log1pexp_exact(double big, double d) {
  const double a = log1pexp_neg(d);
  const double s = big + a;
  const double bb = s - big;
  const double err = (big - (s - bb)) + (a - bb);  // exact residual of the sum
  const double half_ulp = s == 0.0 ? 0.0 : ldexp(1.0, ilogb(s) - 53);
  if (fabs(err) + 4e-16 < half_ulp) return s;
  return big + log1pexp_cr(d);
}

// numpy's npy_logaddexp: the fold np.logaddexp.reduceat performs when the
// reference merges candidates (decoder.py:611) and flag variants (:791).
// EXACT rounds the log1p(exp) term correctly where it matters (see above).
template <bool EXACT = false>
__device__ __forceinline__ double np_logaddexp(double x, double y) {
  if (x == y) return x + CTCB_LN2;
  double tmp = x - y;
  if (tmp > 0) return EXACT ? add_log1pexp_exact(x, tmp) : x + log1pexp_neg(tmp);
  if (tmp <= 0) return EXACT ? add_log1pexp_exact(y, -tmp) : y + log1pexp_neg(-tmp);
  return tmp;
}

// Candidate merge of the reference (decoder.py:610-613, :789-791): logadd
// (numpy's left fold) or max (merge_mode="max").
__device__ __forceinline__ double merge2(double x, double y, bool mx) {
  return mx ? (x > y ? x : y) : np_logaddexp<false>(x, y);
}
__device__ __forceinline__ double merge2_exact(double x, double y, bool mx) {
  return mx ? (x > y ? x : y) : np_logaddexp<true>(x, y);
}

// ---------------------------------------------------------------- prefixes
// Content-defined prefix identity: a chained 64-bit hash of the token
// sequence (plus its length, compared alongside).  The reference interns
// prefixes globally per utterance through child_table (decoder.py:700-711),
// so two hypotheses share a merge key iff their token sequences are equal;
// a chained hash reproduces that equivalence (collision odds ~n^2/2^64).
constexpr uint64_t kEmptyPrefixHash = 0x9e3779b97f4a7c15ull;
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30; x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27; x *= 0x94d049bb133111ebull;
  x ^= x >> 31; return x;
}
__device__ __forceinline__ uint64_t child_hash(uint64_t h, int token) {
  return mix64(h ^ ((uint64_t)(token + 1) * 0xd6e8feb86659fd93ull));
}

// Trellis back-pointer record: source slot (10 bits) | appended token + 1 (22 bits).
constexpr int kSrcShift = 22;
constexpr uint32_t kTokMask = (1u << kSrcShift) - 1;
__device__ __forceinline__ uint32_t pack_trel(int src, int tok) {
  return ((uint32_t)src << kSrcShift) | (uint32_t)(tok + 1);
}
__device__ __forceinline__ int trel_src(uint32_t r) { return (int)(r >> kSrcShift); }
__device__ __forceinline__ int trel_tok(uint32_t r) { return (int)(r & kTokMask) - 1; }

// ---------------------------------------------------------------- input validation
// EmissionMatrix.__post_init__ (emissions.py:128-150) per utterance: any
// non-finite value (code 1), else any value > MAX_LOG_PROB = 1e-4 (code 2),
// else (strict) a row whose fp64 log-sum-exp is off 0 by more than
// ROW_NORM_TOL = 1e-3 (code 3); the first offender in (frame, token) order.
// Key = code << 62 | frame << 30 | (token + 1): the smallest key of an
// utterance is the reference's error.  No float lies in (1e-4f, 1e-4], so the
// fp32 comparison x > 1e-4f equals the reference's fp64 one.
__device__ __forceinline__ unsigned long long vkey_make(int code, int t, int v) {
  return ((unsigned long long)code << 62) | ((unsigned long long)(unsigned)t << 30) | (unsigned long long)(v + 1);
}
// Exact check of one row by a warp: the smallest key of row `t`, or ~0
// (cold path, kept out of line).
static __device__ __noinline__ unsigned long long row_check_exact(const float* row, int V, int t, int lane, bool strict) {
  int v1 = 0x7fffffff, v2 = 0x7fffffff;
  float mx = -INFINITY;
  for (int v = lane; v < V; v += 32) {
    const float x = row[v];
    if (!isfinite(x)) v1 = min(v1, v);
    else if (x > 1e-4f) v2 = min(v2, v);
    mx = fmaxf(mx, x);
  }
  v1 = __reduce_min_sync(0xffffffffu, v1);
  if (v1 != 0x7fffffff) return vkey_make(1, t, v1);
  v2 = __reduce_min_sync(0xffffffffu, v2);
  if (v2 != 0x7fffffff) return vkey_make(2, t, v2);
  if (!strict) return ~0ull;
#pragma unroll
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const double m = (double)mx;
  double sum = 0.0;
  for (int v = lane; v < V; v += 32) sum += exp((double)row[v] - m);
#pragma unroll
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  return fabs(m + log(sum)) > 1e-3 ? vkey_make(3, t, -1) : ~0ull;
}
// Producer/consumer flags between the overlapped top-k kernel and the walk
// (gpu scope), and the programmatic-dependent-launch controls.
__device__ __forceinline__ uint32_t ld_acquire_gpu(const uint32_t* p) {
  uint32_t r;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(r) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait_primary() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Diagnostics: SM id and the global nanosecond timer.
__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long r;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(r));
  return r;
}
// Fast screen of a staged row, split so that the decode kernels keep it off
// their per-frame critical path: row_partials is lane-local (float4 chunks
// c4 = lane, lane + 32, ...), row_verdict (three independent REDUX ops) runs
// later in the frame.  A row passes when it is finite, <= 1e-4 and, if
// strict, the fp32 sum of exp(x) -- in 2^-25 fixed point per lane, clamped at
// 2 -- has |log| < 9e-4; the screen's error is < 1e-4 for V <= 2048, so rows
// near the 1e-3 limit take row_check_exact.
struct RowPart {
  uint32_t kmx, kmn, sfx;
};
__device__ __forceinline__ float ex2_ftz(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// MAXCH: float4 chunks per lane the caller guarantees (4 for V <= 512), 0 = any.
// WITH_MAX = false: the caller folds the row maximum into kmx itself.
// PADDED: the staged row is padded to 4 * MAXCH * 32 floats with -FLT_MAX
// (neutral for every partial), so no chunk needs a bounds check.
template <int MAXCH = 0, bool WITH_MAX = true, bool PADDED = false>
__device__ __forceinline__ RowPart row_partials(const float* row, int V, int lane) {
  const float4* r4 = (const float4*)row;
  constexpr float kL2E = 1.4426950408889634f;
  const float2 l2e2 = make_float2(kL2E, kL2E);
  float2 s2 = make_float2(0.0f, 0.0f);  // packed fp32x2 (FMUL2 / FADD2): half the scale and sum instructions
  float mn = INFINITY, mx = -INFINITY;
  const int nch4 = (V + 3) >> 2;
  const bool ragged = (V & 3) != 0;
  auto chunk = [&](int c4) {
    float4 q = r4[c4];
    if (!PADDED && ragged && 4 * c4 + 4 > V) {  // tail chunk: neutral values past V
      const int c = 4 * c4;
      if (c + 1 >= V) q.y = -1e30f;
      if (c + 2 >= V) q.z = -1e30f;
      if (c + 3 >= V) q.w = -1e30f;
    }
    mn = fminf(mn, fminf(fminf(q.x, q.y), fminf(q.z, q.w)));
    if (WITH_MAX) mx = fmaxf(mx, fmaxf(fmaxf(q.x, q.y), fmaxf(q.z, q.w)));
    const float2 a = __fmul2_rn(make_float2(q.x, q.y), l2e2), b = __fmul2_rn(make_float2(q.z, q.w), l2e2);
    s2 = __fadd2_rn(s2, __fadd2_rn(make_float2(ex2_ftz(a.x), ex2_ftz(a.y)), make_float2(ex2_ftz(b.x), ex2_ftz(b.y))));  // NaN propagates
  };
  if (MAXCH > 0) {
#pragma unroll
    for (int j = 0; j < MAXCH; j++)
      if (PADDED || lane + 32 * j < nch4) chunk(lane + 32 * j);
  } else {
    for (int c4 = lane; c4 < nch4; c4 += 32) chunk(c4);
  }
  const float s = s2.x + s2.y;
  RowPart r;
  r.kmx = s <= 2.0f ? (WITH_MAX ? ord32(mx) : 0u) : 0xffffffffu;  // NaN / huge sums fail the max test
  r.kmn = ord32(mn);
  r.sfx = (uint32_t)(fminf(s, 2.0f) * 33554432.0f);
  return r;
}
__device__ __forceinline__ bool row_verdict(const RowPart& r, bool strict) {
  const uint32_t kmx = __reduce_max_sync(0xffffffffu, r.kmx), kmn = __reduce_min_sync(0xffffffffu, r.kmn);
  const uint32_t sfx = __reduce_add_sync(0xffffffffu, r.sfx);
  const bool ok = kmx <= ord32(1e-4f) && kmn > ord32(-INFINITY);
  // |log(sum)| < 9e-4 as integer bounds on the 2^-25 fixed-point sum:
  // exp(-9e-4) * 2^25 < sfx < exp(9e-4) * 2^25 (no log, no conversion)
  constexpr uint32_t kLo = 33524247u, kHi = 33584644u;
  return ok && (!strict || (sfx > kLo && sfx < kHi));
}
__device__ __forceinline__ bool row_screen(const float* row, int V, int lane, bool strict) {
  return row_verdict(row_partials(row, V, lane), strict);
}
// The same screen over a row in global memory (any alignment).
__device__ __forceinline__ bool row_screen_scalar(const float* row, int V, int lane, bool strict) {
  float s = 0.0f, mn = INFINITY, mx = -INFINITY;
  for (int v = lane; v < V; v += 32) {
    const float x = __ldg(row + v);
    mn = fminf(mn, x);
    mx = fmaxf(mx, x);
    s += __expf(x);
  }
  const uint32_t kmx = __reduce_max_sync(0xffffffffu, ord32(mx)), kmn = __reduce_min_sync(0xffffffffu, ord32(mn));
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const bool ok = kmx <= ord32(1e-4f) && kmn > ord32(-INFINITY) && isfinite(s);
  return ok && (!strict || fabsf(__logf(s)) < 9e-4f);
}

// Python tuple order of seq(ea) + [xa] vs seq(eb) + [xb] (x < 0: no extra
// token) for two entries of a beam after `steps` frames (exact-tie slow path,
// one lane).  Both trellis paths are walked back in lockstep until they reach
// the same entry: everything before it is a common prefix, so only the two
// tails (collected last token first into A / Bq, T_max + 1 ints each) are
// compared.  rec(i, slot) -> {token or -1, source slot} of frame i's record.
// *strict: the sequences differ before the shorter one ends.
template <class Rec>
__device__ __forceinline__ int trellis_seq_cmp(Rec rec, int steps, int ea, int xa, int eb, int xb, int* A, int* Bq,
                                               bool* strict, unsigned long long* dbg) {
  int la = 0, lb = 0;
  if (xa >= 0) A[la++] = xa;
  if (xb >= 0) Bq[lb++] = xb;
  int sa = ea, sb = eb, i = steps - 1;
  for (; i >= 0 && sa != sb; --i) {
    const int2 ra = rec(i, sa), rb = rec(i, sb);
    if (ra.x >= 0) A[la++] = ra.x;
    if (rb.x >= 0) Bq[lb++] = rb.x;
    sa = ra.y;
    sb = rb.y;
  }
  if (dbg) {
    atomicAdd(&dbg[2], 2ull);                                      // kDbgMaterialize
    atomicAdd(&dbg[3], 2ull * (unsigned long long)(steps - 1 - i));  // kDbgMatSteps
  }
  const int n = la < lb ? la : lb;
  *strict = true;
  for (int q = 1; q <= n; q++) {
    const int x = A[la - q], y = Bq[lb - q];
    if (x != y) return x < y ? -1 : 1;
  }
  *strict = false;
  return la < lb ? -1 : (la > lb ? 1 : 0);
}

// ---------------------------------------------------------------- warp
__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---------------------------------------------------------------- token selection
// beam_size_token = K < V (decoder.py:440-458): the K best tokens of the whole
// row, blank included, by (log-prob desc, index asc).  kth_token finds the
// K-th of them as (order key tv, index ti) with an 8-bit radix select on
// ord32 keys (hist: 256 words of shared memory) followed by an index-ordered
// scan of the ties; token c is selected iff ord32(v_c) > tv, or == tv and
// c <= ti.  `row` may hold a sentinel at `blank`: its value is passed as ebf.
// Whole warp, FULL mask.
__device__ __forceinline__ void kth_token(const float* row, int V, int blank, float ebf, int K, uint32_t* hist,
                                          int lane, uint32_t& tv, int& ti) {
  uint32_t prefix = 0, pmask = 0;
  int need = K;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int b = lane; b < 256; b += 32) hist[b] = 0;
    __syncwarp();
    for (int c = lane; c < V; c += 32) {
      const uint32_t key = ord32(c == blank ? ebf : row[c]);
      if ((key & pmask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncwarp();
    uint32_t h[8], sum = 0;
#pragma unroll
    for (int q = 0; q < 8; q++) { h[q] = hist[lane * 8 + q]; sum += h[q]; }
    uint32_t incl = sum;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const uint32_t v = __shfl_down_sync(FULL, incl, off);
      if (lane + off < 32) incl += v;
    }
    uint32_t cum = incl - sum;  // tokens in digits owned by higher lanes
    int found = -1;
    uint32_t cgt = 0;
#pragma unroll
    for (int q = 7; q >= 0; q--) {
      if (found < 0 && cum < (uint32_t)need && cum + h[q] >= (uint32_t)need) { found = lane * 8 + q; cgt = cum; }
      cum += h[q];
    }
    const unsigned bal = __ballot_sync(FULL, found >= 0);
    const int src = __ffs(bal) - 1;
    const int digit = __shfl_sync(FULL, found, src);
    cgt = __shfl_sync(FULL, cgt, src);
    need -= (int)cgt;
    prefix |= (uint32_t)digit << shift;
    pmask |= 0xffu << shift;
    __syncwarp();
  }
  tv = prefix;
  // the need-th token (index order) among those with key == tv
  ti = V - 1;
  for (int c0 = 0; c0 < V; c0 += 32) {
    const int c = c0 + lane;
    const bool eq = c < V && ord32(c == blank ? ebf : row[c]) == tv;
    const unsigned beq = __ballot_sync(FULL, eq);
    const int n = __popc(beq);
    if (need <= n) {
      unsigned m = beq;
      for (int i = 1; i < need; i++) m &= m - 1u;
      ti = c0 + __ffs(m) - 1;
      break;
    }
    need -= n;
  }
}
__device__ __forceinline__ bool token_selected(uint32_t key, int c, uint32_t tv, int ti) {
  return key > tv || (key == tv && c <= ti);
}

// ---------------------------------------------------------------- TMA bulk copy
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// 1-D bulk copy global -> shared through the TMA engine (UBLKCP), completing
// on the mbarrier's transaction count.  dst/src 16 B aligned, bytes % 16 == 0.
__device__ __forceinline__ void tma_bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

}  // namespace ctcb

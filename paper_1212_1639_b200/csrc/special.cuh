// Special functions on the particle path.
//
//  * ndtri   -- standard-normal quantile.  The reference calls
//               scipy.special.ndtri (rng.py:223-224), whose algorithm is the
//               Cephes rational approximation; it is restated here with the
//               same constants and the same un-fused operation order, so the
//               central region (no log) is bit-identical to scipy and the
//               tails differ only where CUDA's log() and glibc's log() round
//               differently.
//  * gamma_quantile_accurate -- the Gamma(a,1) quantile the reference takes
//               from scipy.special.gammaincinv (rng.py:226-229,
//               filtering.py:280,286): Halley iteration on the regularized
//               incomplete gamma function with a cancellation-free prefactor.
//               Used to build tables and as the slow "accurate" draw method.
//  * gamma_table_eval -- the hot-path draw.  The shape a_t = a0 + t/2 is
//               the same for every particle in a step (filtering.py:279,285),
//               so each step gets a piecewise-polynomial table of u -> g in
//               u-space: 51 binades x 4 sub-segments per tail plus 32 central
//               segments, degree 11 (Horner with FMA).  No transcendental on
//               the draw path.
//  * nt_eval -- the hot-path normal draw: the same u-space piecewise table
//               for ndtri on v = min(u, 1-u) (ndtri is odd about 1/2), the
//               central quarter fitted as ndtri(v)/(v - 1/2) so relative
//               accuracy holds down to the zero.  Branch-free apart from
//               the segment index, so a warp no longer executes both the
//               central and the log/sqrt tail branch of the Cephes code.
#pragma once
#include <math.h>

#include "common.cuh"

namespace pf {

// ------------------------------------------------------------------ ndtri --
__host__ __device__ inline double polevl_(double x, const double* c, int n) {
  double a = c[0];
  for (int i = 1; i <= n; ++i) a = a * x + c[i];
  return a;
}
__host__ __device__ inline double p1evl_(double x, const double* c, int n) {
  double a = x + c[0];
  for (int i = 1; i < n; ++i) a = a * x + c[i];
  return a;
}

PF_HD double ndtri(double y0) {
  const double s2pi = 2.50662827463100050242E0;
  const double expm2 = 0.13533528323661269189;
  const double P0[5] = {-5.99633501014107895267E1, 9.80010754185999661536E1,
                        -5.66762857469070293439E1, 1.39312609387279679503E1,
                        -1.23916583867381258016E0};
  const double Q0[8] = {1.95448858338141759834E0,  4.67627912898881538453E0,
                        8.63602421390890590575E1,  -2.25462687854119370527E2,
                        2.00260212380060660359E2,  -8.20372256168333339912E1,
                        1.59056225126211695515E1,  -1.18331621121330003142E0};
  const double P1[9] = {4.05544892305962419923E0,   3.15251094599893866154E1,
                        5.71628192246421288162E1,   4.40805073893200834700E1,
                        1.46849561928858024014E1,   2.18663306850790267539E0,
                        -1.40256079171354495875E-1, -3.50424626827848203418E-2,
                        -8.57456785154685413611E-4};
  const double Q1[8] = {1.57799883256466749731E1,   4.53907635128879210584E1,
                        4.13172038254672030440E1,   1.50425385692907503408E1,
                        2.50464946208309415979E0,   -1.42182922854787788574E-1,
                        -3.80806407691578277194E-2, -9.33259480895457427372E-4};
  const double P2[9] = {3.23774891776946035970E0,  6.91522889068984211695E0,
                        3.93881025292474443415E0,  1.33303460815807542389E0,
                        2.01485389549179081538E-1, 1.23716634817820021358E-2,
                        3.01581553508235416007E-4, 2.65806974686737550832E-6,
                        6.23974539184983293730E-9};
  const double Q2[8] = {6.02427039364742014255E0,  3.67983563856160859403E0,
                        1.37702099489081330271E0,  2.16236993594496635890E-1,
                        1.34204006088543189037E-2, 3.28014464682127739104E-4,
                        2.89247864745380683936E-6, 6.79019408009981274425E-9};
  if (y0 <= 0.0) return -INFINITY;
  if (y0 >= 1.0) return INFINITY;
  int code = 1;
  double y = y0;
  if (y > (1.0 - expm2)) {
    y = 1.0 - y;
    code = 0;
  }
  if (y > expm2) {
    y = y - 0.5;
    double y2 = y * y;
    double x = y + y * (y2 * polevl_(y2, P0, 4) / p1evl_(y2, Q0, 8));
    return x * s2pi;
  }
  double x = sqrt(-2.0 * log(y));
  double x0 = x - log(x) / x;
  double z = 1.0 / x;
  double x1;
  if (x < 8.0)
    x1 = z * polevl_(z, P1, 8) / p1evl_(z, Q1, 8);
  else
    x1 = z * polevl_(z, P2, 8) / p1evl_(z, Q2, 8);
  x = x0 - x1;
  if (code != 0) x = -x;
  return x;
}

// ---------------------------------------------------- incomplete gamma ----
// log(1+d) - d without cancellation.
PF_HD double log1pmx(double d) {
  if (fabs(d) < 0.25) {
    double dk = d * d, sum = 0.0;
    for (int k = 2; k < 80; ++k) {
      double t = dk / k;
      sum += (k & 1) ? t : -t;
      if (fabs(t) <= 1e-19 * fabs(sum)) break;
      dk *= d;
    }
    return sum;
  }
  return log1p(d) - d;
}

// log of D(a,x) = x^a e^-x / Gamma(a+1).  Stirling form for a >= 10 keeps
// a*log(x) - x from cancelling against lgamma.
PF_HD double log_gamma_prefactor(double a, double x) {
  if (a < 10.0) return a * log(x) - x - lgamma(a + 1.0);
  const double LOG_2PI = 1.8378770664093454836;
  double ia = 1.0 / a, ia2 = ia * ia;
  // Stirling correction eps(a) of lgamma(a+1) = (a+1/2)log a - a + log(2pi)/2 + eps
  double eps = ia * (1.0 / 12 + ia2 * (-1.0 / 360 + ia2 * (1.0 / 1260 + ia2 * (-1.0 / 1680 +
              ia2 * (1.0 / 1188 + ia2 * (-691.0 / 360360 + ia2 * (1.0 / 156)))))));
  double d = (x - a) / a;
  return a * log1pmx(d) - 0.5 * (LOG_2PI + log(a)) - eps;
}

// Regularized P(a,x) (lower=true) or Q(a,x) (lower=false); also returns D.
PF_HD double gamma_pq(double a, double x, bool lower, double* dprefac) {
  double lD = log_gamma_prefactor(a, x);
  double D = exp(lD);
  if (dprefac) *dprefac = D;
  if (x <= 0.0) return lower ? 0.0 : 1.0;
  if (x < a + 1.0) {
    double sum = 1.0, term = 1.0;
    for (int n = 1; n < 100000; ++n) {
      term *= x / (a + n);
      sum += term;
      if (term < sum * 1e-17) break;
    }
    double P = D * sum;
    return lower ? P : 1.0 - P;
  }
  // Lentz continued fraction for Q (x >= a+1).
  const double FPMIN = 1e-300;
  double b = x + 1.0 - a, c = 1.0 / FPMIN, dd = 1.0 / b, h = dd;
  for (int i = 1; i < 100000; ++i) {
    double an = -i * (i - a);
    b += 2.0;
    dd = an * dd + b;
    if (fabs(dd) < FPMIN) dd = FPMIN;
    c = b + an / c;
    if (fabs(c) < FPMIN) c = FPMIN;
    dd = 1.0 / dd;
    double del = dd * c;
    h *= del;
    if (fabs(del - 1.0) < 4e-16) break;  // del == 1 to within an ulp
  }
  double Q = D * a * h;
  return lower ? 1.0 - Q : Q;
}

// Gamma(a,1) quantile: P(a,x) = u for u <= 1/2, else Q(a,x) = v with the
// exact complement v = 1 - u supplied (so upper tails keep full accuracy).
PF_HD double gamma_quantile_pv(double a, double p, double v, bool lower) {
  // Wilson-Hilferty start, repaired for small shapes / extreme tails.
  double z = lower ? ndtri(p) : -ndtri(v);
  double x;
  double s = 1.0 / (9.0 * a);
  double wh = 1.0 - s + z * sqrt(s);
  x = a * wh * wh * wh;
  if (!(x > 0.0) || a < 1.0) {
    if (lower)
      x = exp((log(p) + lgamma(a + 1.0)) / a);  // P ~ x^a / Gamma(a+1)
    else
      x = fmax(a, -log(v) + (a - 1.0) * log(fmax(1.0, -log(v))));
  }
  double lo = 0.0, hi = INFINITY;
  double last_step = INFINITY;
  for (int it = 0; it < 80; ++it) {
    double D;
    double f = gamma_pq(a, x, lower, &D);
    double F = lower ? (f - p) : (v - f);  // increasing in x
    if (F == 0.0) return x;
    if (F > 0.0) hi = x; else lo = x;
    double dF = D * a / x;  // d/dx P(a,x)
    double r = F / dF;
    double h2 = (a - 1.0) / x - 1.0;  // F''/F'
    double den = 1.0 - 0.5 * r * h2;
    double step = (den > 0.5 && den < 2.0) ? r / den : r;
    double xn = x - step;
    if (!(xn > lo && xn < hi) || !(dF > 0.0)) {
      xn = (hi == INFINITY) ? (lo > 0 ? lo * 2.0 : x * 2.0) : (lo > 0.0 ? sqrt(lo * hi) : 0.5 * hi);
    }
    const double dx = fabs(xn - x);
    // converged to an ulp, or Halley has started to oscillate at rounding level
    if (dx <= 4e-16 * x || (it > 3 && dx >= last_step && dx <= 1e-13 * x)) {
      x = xn;
      break;
    }
    last_step = dx;
    x = xn;
  }
  return x;
}

PF_HD double gamma_quantile_accurate(double a, double u) {
  if (u <= 0.5) return gamma_quantile_pv(a, u, 1.0 - u, true);
  return gamma_quantile_pv(a, u, 1.0 - u, false);
}

// --------------------------------------------------------- per-step table --
constexpr int GT_SUB = 4;                       // sub-segments per binade
constexpr int GT_BINADES = 51;                  // exponents -53..-3
constexpr int GT_TAIL = GT_BINADES * GT_SUB;    // 204 segments per tail
constexpr int GT_CENTRAL = 32;                  // uniform segments on [1/4, 3/4]
constexpr int GT_NSEG = 2 * GT_TAIL + GT_CENTRAL;  // 440
constexpr int GT_DEG = 11;
constexpr int GT_NC = GT_DEG + 1;               // 12 coefficients (96 B / segment)
constexpr int GT_TABLE_DOUBLES = GT_NSEG * GT_NC;

// Segment and local coordinate t in [-1,1] of a uniform u in (0,1).  Also
// used to place the Chebyshev nodes when the table is built, so evaluation
// and construction agree by construction.
PF_HD int gt_segment(double u, double* t) {
  union { double d; uint64_t b; } c;
  if (u < 0.25 || u > 0.75) {
    bool up = u > 0.75;
    double v = up ? 1.0 - u : u;  // exact for u > 3/4
    c.d = v;
    int e = int((c.b >> 52) & 0x7FF) - 1023;  // v in [2^e, 2^(e+1))
    if (e < -53) e = -53;
    int i = int((c.b >> (52 - 2)) & 3);
    c.b = (c.b & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull;  // mantissa in [1,2)
    *t = (c.d - (1.0 + (i + 0.5) * 0.25)) * 8.0;
    int seg = (e + 53) * GT_SUB + i;
    return up ? GT_TAIL + GT_CENTRAL + seg : seg;
  }
  double xx = (u - 0.25) * (2.0 * GT_CENTRAL);
  int j = int(xx);
  if (j > GT_CENTRAL - 1) j = GT_CENTRAL - 1;
  *t = (xx - j - 0.5) * 2.0;
  return GT_TAIL + j;
}

// Branch-free gt_segment for the hot path: both the tail and the central
// coordinates are formed with the same operations as gt_segment and the
// result is selected, so (seg, t) are identical -- but a warp whose lanes
// straddle u = 1/4 or 3/4 no longer executes the two paths one after the
// other, and the three draws of a slot stay in one basic block.
PF_HD int gt_segment_bf(double u, double* t) {
  union { double d; uint64_t b; } c;
  const bool up = u > 0.5;
  const double v = up ? 1.0 - u : u;  // exact for u > 1/2; equals gt_segment's v in the tails
  c.d = v;
  int e = int((c.b >> 52) & 0x7FF) - 1023;
  e = e < -53 ? -53 : e;
  const int i = int((c.b >> (52 - 2)) & 3);
  c.b = (c.b & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull;
  const double tt = (c.d - (1.0 + (i + 0.5) * 0.25)) * 8.0;
  const int st = (e + 53) * GT_SUB + i;
  const double xx = (u - 0.25) * (2.0 * GT_CENTRAL);
  int j = int(xx);
  j = j < 0 ? 0 : (j > GT_CENTRAL - 1 ? GT_CENTRAL - 1 : j);
  const double tc = (xx - j - 0.5) * 2.0;
  const bool tail = u < 0.25 || u > 0.75;
  *t = tail ? tt : tc;
  return tail ? (up ? GT_TAIL + GT_CENTRAL + st : st) : GT_TAIL + j;
}

// Inverse of gt_segment: the uniform (and, for the upper tail, its exact
// complement) at local coordinate t of segment seg.
PF_HD void gt_point(int seg, double t, double* u, double* v, bool* upper) {
  if (seg >= GT_TAIL && seg < GT_TAIL + GT_CENTRAL) {
    int j = seg - GT_TAIL;
    *u = 0.25 + (j + 0.5 + 0.5 * t) / (2.0 * GT_CENTRAL);
    *v = 1.0 - *u;
    *upper = *u > 0.5;
    return;
  }
  bool up = seg >= GT_TAIL + GT_CENTRAL;
  int s = up ? seg - GT_TAIL - GT_CENTRAL : seg;
  int e = s / GT_SUB - 53, i = s % GT_SUB;
  double m = 1.0 + (i + 0.5 + 0.5 * t) * 0.25;
  double w = ldexp(m, e);
  if (up) {
    *v = w;
    *u = 1.0 - w;
    *upper = true;
  } else {
    *u = w;
    *v = 1.0 - w;
    *upper = false;
  }
}

template <typename CoefPtr>
PF_HD double gt_eval(CoefPtr coef, double u) {
  double t;
  int seg = gt_segment(u, &t);
  const double* c = &coef[seg * GT_NC];
  double r = c[GT_DEG];
#pragma unroll
  for (int k = GT_DEG - 1; k >= 0; --k) r = fma(r, t, c[k]);
  return r;
}

// --------------------------------------------------- normal quantile table --
constexpr int NT_TAIL = GT_BINADES * GT_SUB;    // v in [2^-53, 1/4): 204 segments
constexpr int NT_CENTRAL = 16;                  // v in [1/4, 1/2]
constexpr int NT_NSEG = NT_TAIL + NT_CENTRAL;   // 220
constexpr int NT_TABLE_DOUBLES = NT_NSEG * GT_NC;

// Segment of u, local coordinate t in [-1,1], and the factor the table
// polynomial is multiplied by (sign; (v - 1/2) in the central segments).
PF_HD int nt_segment(double u, double* t, double* scale) {
  const bool up = u > 0.5;
  const double v = up ? 1.0 - u : u;  // exact for u >= 1/2
  const double sg = up ? -1.0 : 1.0;
  if (v < 0.25) {
    union { double d; uint64_t b; } c;
    c.d = v;
    int e = int((c.b >> 52) & 0x7FF) - 1023;
    if (e < -53) e = -53;
    const int i = int((c.b >> (52 - 2)) & 3);
    c.b = (c.b & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull;
    *t = (c.d - (1.0 + (i + 0.5) * 0.25)) * 8.0;
    *scale = sg;
    return (e + 53) * GT_SUB + i;
  }
  const double xx = (v - 0.25) * (4.0 * NT_CENTRAL);
  int j = int(xx);
  if (j > NT_CENTRAL - 1) j = NT_CENTRAL - 1;
  *t = (xx - j - 0.5) * 2.0;
  *scale = sg * (v - 0.5);  // exact
  return NT_TAIL + j;
}

// Branch-free nt_segment (same operations, selected): identical (seg, t,
// scale), no divergence between tail and central lanes.
PF_HD int nt_segment_bf(double u, double* t, double* scale) {
  const bool up = u > 0.5;
  const double v = up ? 1.0 - u : u;  // exact for u >= 1/2
  const double sg = up ? -1.0 : 1.0;
  union { double d; uint64_t b; } c;
  c.d = v;
  int e = int((c.b >> 52) & 0x7FF) - 1023;
  e = e < -53 ? -53 : e;
  const int i = int((c.b >> (52 - 2)) & 3);
  c.b = (c.b & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull;
  const double tt = (c.d - (1.0 + (i + 0.5) * 0.25)) * 8.0;
  const double xx = (v - 0.25) * (4.0 * NT_CENTRAL);
  int j = int(xx);
  j = j < 0 ? 0 : (j > NT_CENTRAL - 1 ? NT_CENTRAL - 1 : j);
  const double tc = (xx - j - 0.5) * 2.0;
  const bool tail = v < 0.25;
  *t = tail ? tt : tc;
  *scale = tail ? sg : sg * (v - 0.5);  // exact
  return tail ? (e + 53) * GT_SUB + i : NT_TAIL + j;
}

// The v (<= 1/2) at local coordinate t of segment seg, and whether the
// segment is central (fitted as ndtri(v)/(v-1/2)).
PF_HD double nt_point(int seg, double t, bool* central) {
  if (seg >= NT_TAIL) {
    *central = true;
    return 0.25 + (seg - NT_TAIL + 0.5 + 0.5 * t) / (4.0 * NT_CENTRAL);
  }
  *central = false;
  const int e = seg / GT_SUB - 53, i = seg % GT_SUB;
  return ldexp(1.0 + (i + 0.5 + 0.5 * t) * 0.25, e);
}

template <typename CoefPtr>
PF_HD double nt_eval(CoefPtr coef, double u) {
  double t, sc;
  const int seg = nt_segment(u, &t, &sc);
  const double* c = &coef[seg * GT_NC];
  double r = c[GT_DEG];
#pragma unroll
  for (int k = GT_DEG - 1; k >= 0; --k) r = fma(r, t, c[k]);
  return sc * r;
}

// Chebyshev interpolant through f at the GT_NC Chebyshev nodes of [-1,1],
// converted to monomial coefficients in t (one thread).  Coefficients below
// trunc * max|f| are rounding noise of the DCT; the monomial expansion would
// amplify them (T_11 has coefficients up to 2^10), so they are dropped.
PF_HD void cheb_to_mono(const double* f, double* out, double trunc = 0.0) {
  const double PI = 3.14159265358979323846;
  double c[GT_NC];
  for (int k = 0; k < GT_NC; ++k) {
    double s = 0.0;
    for (int i = 0; i < GT_NC; ++i) s += f[i] * cos(PI * k * (i + 0.5) / GT_NC);
    c[k] = s * (2.0 / GT_NC);
  }
  c[0] *= 0.5;
  if (trunc > 0.0) {
    double fm = 0.0;
    for (int i = 0; i < GT_NC; ++i) fm = fmax(fm, fabs(f[i]));
    for (int k = 1; k < GT_NC; ++k)
      if (fabs(c[k]) < trunc * fm) c[k] = 0.0;
  }
  double tm[GT_NC] = {0}, tk[GT_NC] = {0}, mono[GT_NC] = {0};
  tm[0] = 1.0;
  tk[1] = 1.0;
  mono[0] = c[0];
  for (int i = 0; i < GT_NC; ++i) mono[i] += c[1] * tk[i];
  for (int k = 2; k < GT_NC; ++k) {
    double tn[GT_NC];
    for (int i = 0; i < GT_NC; ++i) tn[i] = (i ? 2.0 * tk[i - 1] : 0.0) - tm[i];
    for (int i = 0; i < GT_NC; ++i) {
      mono[i] += c[k] * tn[i];
      tm[i] = tk[i];
      tk[i] = tn[i];
    }
  }
  for (int i = 0; i < GT_NC; ++i) out[i] = mono[i];
}

}  // namespace pf

/* TEST INFRASTRUCTURE ONLY -- CPU oracle backend; see r2r.h. */
#include "r2r.h"

#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  double re, im;
} cpx;

static const double PI = 3.14159265358979323846264338327950288;

/* ---- power-of-two complex FFT (iterative radix-2, exact twiddles) ---- */
typedef struct {
  size_t p;
  cpx* tw;       /* p/2 twiddles e^{-2 pi i k / p} */
  size_t* rev;   /* bit reversal */
} fftplan;

static void fft_init(fftplan* f, size_t p) {
  f->p = p;
  f->tw = (cpx*)malloc(sizeof(cpx) * (p / 2 + 1));
  f->rev = (size_t*)malloc(sizeof(size_t) * p);
  for (size_t k = 0; k < p / 2; ++k) {
    /* angle reduced exactly: 2 pi k / p */
    const double a = 2.0 * PI * (double)k / (double)p;
    f->tw[k].re = cos(a);
    f->tw[k].im = -sin(a);
  }
  int lg = 0;
  while (((size_t)1 << lg) < p) ++lg;
  for (size_t i = 0; i < p; ++i) {
    size_t r = 0;
    for (int b = 0; b < lg; ++b)
      if (i & ((size_t)1 << b)) r |= (size_t)1 << (lg - 1 - b);
    f->rev[i] = r;
  }
}

/* sign = -1 forward (e^{-i}), +1 inverse (e^{+i}), unnormalised */
static void fft_run(const fftplan* f, cpx* a, int sign) {
  const size_t p = f->p;
  for (size_t i = 0; i < p; ++i) {
    const size_t r = f->rev[i];
    if (r > i) {
      cpx t = a[i];
      a[i] = a[r];
      a[r] = t;
    }
  }
  for (size_t len = 2; len <= p; len <<= 1) {
    const size_t half = len >> 1, step = p / len;
    for (size_t s = 0; s < p; s += len) {
      for (size_t j = 0; j < half; ++j) {
        cpx w = f->tw[j * step];
        if (sign > 0) w.im = -w.im;
        cpx* u = &a[s + j];
        cpx* v = &a[s + j + half];
        const double tr = v->re * w.re - v->im * w.im;
        const double ti = v->re * w.im + v->im * w.re;
        v->re = u->re - tr;
        v->im = u->im - ti;
        u->re += tr;
        u->im += ti;
      }
    }
  }
}

/* ---- chirp-z: X_k = sum_{j<m_in} x_j e^{+i pi j k / den}, k < m_out ---- */
typedef struct czt {
  int kind;
  size_t n;
  size_t m_in, m_out, den;
  fftplan f;
  cpx* chirp;  /* e^{+i pi t^2/(2 den)} for t < max(m_in, m_out) */
  cpx* bhat;   /* FFT of e^{-i pi t^2/(2 den)} wrapped */
  cpx* twin;   /* input twiddle (kind-specific), length m_in */
  cpx* twout;  /* output twiddle, length m_out */
  struct czt* next;
} czt;

static cpx expi_pi(uint64_t num, uint64_t den2) {
  /* e^{i pi num / den2} with num reduced mod 2*den2 exactly */
  const uint64_t r = num % (2 * den2);
  const double a = PI * (double)r / (double)den2;
  cpx c = {cos(a), sin(a)};
  return c;
}

static czt* czt_build(int kind, size_t n) {
  czt* z = (czt*)calloc(1, sizeof(czt));
  z->kind = kind;
  z->n = n;
  z->den = n;
  switch (kind) {
    case R2R_REDFT01: z->m_in = n; z->m_out = n; break;
    case R2R_RODFT01: z->m_in = n + 1; z->m_out = n; break;
    case R2R_REDFT10: z->m_in = n; z->m_out = n; break;
    case R2R_RODFT10: z->m_in = n; z->m_out = n + 1; break;
    default: free(z); return NULL;
  }
  size_t p = 1;
  while (p < z->m_in + z->m_out - 1) p <<= 1;
  fft_init(&z->f, p);
  const size_t tmax = z->m_in > z->m_out ? z->m_in : z->m_out;
  z->chirp = (cpx*)malloc(sizeof(cpx) * tmax);
  for (size_t t = 0; t < tmax; ++t) z->chirp[t] = expi_pi((uint64_t)t * t, 2 * (uint64_t)n);
  z->bhat = (cpx*)calloc(p, sizeof(cpx));
  for (size_t t = 0; t < tmax; ++t) {
    cpx c = z->chirp[t];
    c.im = -c.im;
    if (t < z->m_out) z->bhat[t] = c;
    if (t > 0 && t < z->m_in) z->bhat[p - t] = c;
  }
  fft_run(&z->f, z->bhat, -1);
  z->twin = (cpx*)malloc(sizeof(cpx) * z->m_in);
  z->twout = (cpx*)malloc(sizeof(cpx) * z->m_out);
  for (size_t j = 0; j < z->m_in; ++j) {
    if (kind == R2R_REDFT01 || kind == R2R_RODFT01)
      z->twin[j] = expi_pi(j, 2 * (uint64_t)n); /* e^{i pi j /(2n)} */
    else {
      cpx one = {1.0, 0.0};
      z->twin[j] = one;
    }
  }
  for (size_t k = 0; k < z->m_out; ++k) {
    if (kind == R2R_REDFT10 || kind == R2R_RODFT10)
      z->twout[k] = expi_pi(k, 2 * (uint64_t)n); /* e^{i pi k /(2n)} */
    else {
      cpx one = {1.0, 0.0};
      z->twout[k] = one;
    }
  }
  return z;
}

static pthread_mutex_t g_lock = PTHREAD_MUTEX_INITIALIZER;
static czt* g_plans = NULL;

static czt* czt_get(int kind, size_t n) {
  pthread_mutex_lock(&g_lock);
  czt* z = g_plans;
  while (z && !(z->kind == kind && z->n == n)) z = z->next;
  if (!z) {
    z = czt_build(kind, n);
    if (z) {
      z->next = g_plans;
      g_plans = z;
    }
  }
  pthread_mutex_unlock(&g_lock);
  return z;
}

static inline cpx cmul(cpx a, cpx b) {
  cpx c = {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
  return c;
}

int r2r_execute(int kind, size_t n, const double* in, double* out) {
  if (n == 0) return -1;
  czt* z = czt_get(kind, n);
  if (!z) return -1;
  const size_t p = z->f.p;
  cpx* a = (cpx*)calloc(p, sizeof(cpx));
  if (!a) return -1;
  /* real input sequence x_j (j < m_in) */
  for (size_t j = 0; j < z->m_in; ++j) {
    double xj = 0.0;
    switch (kind) {
      case R2R_REDFT01: xj = j == 0 ? in[0] : 2.0 * in[j]; break;
      case R2R_RODFT01: xj = j == 0 ? 0.0 : (j < n ? 2.0 * in[j - 1] : in[n - 1]); break;
      default: xj = in[j]; break;
    }
    cpx v = {xj, 0.0};
    v = cmul(v, z->twin[j]);
    a[j] = cmul(v, z->chirp[j]);
  }
  fft_run(&z->f, a, -1);
  for (size_t i = 0; i < p; ++i) a[i] = cmul(a[i], z->bhat[i]);
  fft_run(&z->f, a, +1);
  const double inv = 1.0 / (double)p;
  for (size_t k = 0; k < z->m_out; ++k) {
    cpx v = a[k];
    v.re *= inv;
    v.im *= inv;
    v = cmul(v, z->chirp[k]);
    v = cmul(v, z->twout[k]);
    switch (kind) {
      case R2R_REDFT01: out[k] = v.re; break;
      case R2R_RODFT01: out[k] = v.im; break;
      case R2R_REDFT10: out[k] = 2.0 * v.re; break;
      case R2R_RODFT10:
        if (k >= 1) out[k - 1] = 2.0 * v.im;
        break;
    }
  }
  free(a);
  return 0;
}

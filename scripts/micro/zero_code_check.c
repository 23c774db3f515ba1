// Host restatement check: the walker's short zero-code predicate equals
// quantize(v, pred) == (radius, not outlier) (run by tests/test_zero_code.py).
#include <math.h>
#include <stdio.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
typedef struct { double eb, two_eb, inv2eb; int radius, use_recip; } QP;
static int quant(double v, double pred, const QP* P, float* rec, int* outl) {
  double d = v - pred, q, aq, f, fr;
  if (P->use_recip) { q = d * P->inv2eb; aq = fabs(q); f = floor(aq); fr = aq - f;
    double tol = aq * 1.7763568394002505e-15 + 1e-300;
    if (fabs(fr - 0.5) <= tol) { q = d / P->two_eb; aq = fabs(q); f = floor(aq); fr = aq - f; }
  } else { q = d / P->two_eb; aq = fabs(q); f = floor(aq); fr = aq - f; }
  double r = (fr >= 0.5) ? f + 1.0 : f;
  if (r < (double)P->radius) { int s = (int)r; if (q < 0.0) s = -s;
    float rc = (float)(pred + P->two_eb * (double)s);
    if (fabs((double)rc - v) <= P->eb) { *rec = rc; *outl = 0; return s + P->radius; } }
  *rec = (float)v; *outl = 1; return P->radius;
}
static int zfull(double v, double pred, const QP* P) { float r; int o; int c = quant(v, pred, P, &r, &o); return c == P->radius && !o; }
static int zfast(double v, double pred, const QP* P) {
  const double d = v - pred; double aq;
  if (P->use_recip) { aq = fabs(d * P->inv2eb); const double tol = aq * 1.7763568394002505e-15 + 1e-300;
    if (fabs(aq - 0.5) <= tol) aq = fabs(d / P->two_eb);
  } else aq = fabs(d / P->two_eb);
  const float rc = (float)(pred + P->two_eb * 0.0);
  return aq < 0.5 && fabs((double)rc - v) <= P->eb && P->radius > 0;
}
static uint64_t s = 88172645463325252ull; static uint64_t xr(void){ s ^= s<<13; s ^= s>>7; s ^= s<<17; return s; }
static float rf(void){ for(;;){ uint32_t u = (uint32_t)xr(); float f; memcpy(&f,&u,4); if (isfinite(f)) return f; } }
int main(void) {
  long bad = 0, n = 0, zc = 0;
  for (int it = 0; it < 200000; it++) {
    QP P; double eb;
    switch (xr() % 4) { case 0: eb = ldexp((double)(xr() % 1000 + 1), -(int)(xr() % 40)); break;
      case 1: eb = fabs((double)rf()); break; case 2: eb = 1e-3; break; default: eb = ldexp(1.0, (int)(xr()%60) - 30); }
    if (!(eb > 0) || !isfinite(eb)) continue;
    P.eb = eb; P.two_eb = 2.0 * eb; P.inv2eb = 1.0 / P.two_eb; P.radius = (xr() % 8 == 0) ? 1 : 512;
    P.use_recip = isfinite(P.inv2eb) && P.two_eb >= 2.2250738585072014e-308;
    float pf = (xr() % 3 == 0) ? rf() : (float)((double)(int32_t)xr() * 1e-6);
    double pred = (double)pf;
    for (int j = 0; j < 200; j++) {
      float vf;
      switch (xr() % 5) {
        case 0: vf = rf(); break;
        case 1: vf = (float)(pred + (((double)(xr() % 2001) - 1000.0) / 1000.0) * 2.0 * eb); break;
        case 2: vf = (float)(pred + ((xr() & 1) ? 1 : -1) * eb); break;   // tie-ish
        case 3: { float b = (float)(pred + ((xr() & 1) ? 1 : -1) * eb); uint32_t u; memcpy(&u,&b,4); u += (int)(xr()%9) - 4; memcpy(&vf,&u,4); break; }
        default: vf = (float)(pred + ((double)(xr() % 7) - 3.0) * 0.5 * 2.0 * eb); break;
      }
      if (!isfinite(vf)) continue;
      int a = zfull(vf, pred, &P), b = zfast(vf, pred, &P); n++; zc += a;
      if (a != b) { if (bad < 10) printf("MISMATCH v=%.17g pred=%.17g eb=%.17g a=%d b=%d\n", (double)vf, pred, eb, a, b); bad++; }
    }
  }
  printf("n=%ld zero=%ld bad=%ld\n", n, zc, bad);
  return bad != 0;
}

// TEST INFRASTRUCTURE: checks a restatement of glibc 2.39 hypot (dbl-64 e_hypot.c,
// non-FMA kernel) bitwise against the host libm; mirrored by ign::ghypot in
// paper_2202_02319_b200/csrc/physics.cuh. Exit status = number of mismatches (capped).
#include <math.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>
#include <stdlib.h>
#define SCALE 0x1p-600
#define LARGE_VAL 0x1p+511
#define TINY_VAL 0x1p-511
#define EPS 0x1p-54
static inline double kernel(double ax, double ay) {
  double t1, t2;
  double h = sqrt(ax * ax + ay * ay);
  if (h <= 2.0 * ay) {
    double delta = h - ay;
    t1 = ax * (2.0 * delta - ax);
    t2 = (delta - 2.0 * (ax - ay)) * delta;
  } else {
    double delta = h - ax;
    t1 = 2.0 * delta * (ax - 2.0 * ay);
    t2 = (4.0 * delta - ay) * ay + delta * delta;
  }
  h -= (t1 + t2) / (2.0 * h);
  return h;
}
double myhypot(double x, double y) {
  if (!isfinite(x) || !isfinite(y)) { if (isinf(x) || isinf(y)) return INFINITY; return x + y; }
  x = fabs(x); y = fabs(y);
  double ax = x < y ? y : x, ay = x < y ? x : y;
  if (ax > LARGE_VAL) { if (ay <= ax * EPS) return ax + ay; return kernel(ax * SCALE, ay * SCALE) / SCALE; }
  if (ay < TINY_VAL) { if (ax >= ay / EPS) return ax + ay; ax = kernel(ax / SCALE, ay / SCALE) * SCALE; return ax; }
  if (ay <= ax * EPS) return ax + ay;
  return kernel(ax, ay);
}
static uint64_t s=88172645463325252ull; static uint64_t xr(){ s^=s<<13; s^=s>>7; s^=s<<17; return s;}
static double rnd(){ uint64_t b = xr(); int e = (int)(xr()%200) - 100; double m = (double)(b>>11)/9007199254740992.0 + 0.5; double v = ldexp(m, e); if (xr()&1) v=-v; return v;}
int main(int argc, char** argv){ long bad=0; long n = argc > 1 ? atol(argv[1]) : 20000000;
 for(long i=0;i<n;++i){ double a=rnd(), b=rnd(); if (i%3==0) b = a*ldexp((double)(xr()>>11)/9007199254740992.0, -(int)(xr()%60));
   double g=hypot(a,b), m=myhypot(a,b); if (memcmp(&g,&m,8)) { if (bad<5) printf("%a %a glibc %a mine %a\n",a,b,g,m); ++bad; } }
 printf("mismatches %ld of %ld\n", bad, n); return bad ? 1 : 0; }

#include <stdio.h>
#include <stdlib.h>
#include <math.h>
#include <stdint.h>
// 1D Lorenzo step (predict.py:70-90 with pred = 0.0 + r)
static inline float step(float r, float xv, double eb, double two_eb, int64_t R, int first) {
    double v = xv, pred = first ? 0.0 : 0.0 + (double)r;
    double q = (v - pred) / two_eb, aq = fabs(q), f = floor(aq);
    double rr = (aq - f >= 0.5) ? f + 1.0 : f;
    if (rr < (double)R) { int64_t s = (int64_t)rr; if (q < 0) s = -s;
        float rec = (float)(pred + two_eb * (double)s);
        if (fabs((double)rec - v) <= eb) return rec; }
    return xv;
}
int main(int argc, char** argv) {
    FILE* f = fopen(argv[1], "rb"); fseek(f, 0, SEEK_END); long n = ftell(f) / 4; fseek(f, 0, SEEK_SET);
    float* x = malloc(n * 4); fread(x, 4, n, f); fclose(f);
    double rel = atof(argv[2]);
    float lo = x[0], hi = x[0]; for (long i = 0; i < n; i++) { if (x[i] < lo) lo = x[i]; if (x[i] > hi) hi = x[i]; }
    double eb = rel * ((double)hi - (double)lo), two_eb = 2 * eb;
    float* tr = malloc(n * 4); float r = 0; long nev = 0;
    for (long i = 0; i < n; i++) { float nr = step(r, x[i], eb, two_eb, 512, i == 0); if (nr != r || i == 0) nev++; r = nr; tr[i] = r; }
    printf("n %ld eb %g events~ %ld\n", n, eb, nev);
    int nc = atoi(argv[3]);
    for (int c = 1; c < nc; c++) {
        long P = n / nc * c;
        for (int g = 0; g < 3; g++) {
            float s = g == 0 ? x[P - 1] : (g == 1 ? nextafterf(tr[P-1], 1e30f) : tr[P-1] + (float)eb * 0.5f);
            long ev = 0, p;
            for (p = P; p < n; p++) { float ns = step(s, x[p], eb, two_eb, 512, 0); if (ns != s) ev++; s = ns; if (s == tr[p]) break; }
            printf("P=%ld guess%d: sync after %ld elems, %ld spec events\n", P, g, p - P, ev);
        }
    }
}

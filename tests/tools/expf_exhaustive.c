/* TEST TOOL: compares the device expf port (sfg_expf.h, compiled for the
 * host) against the host libm expf over all 2^32 float bit patterns.
 * Prints the mismatch count (NaN payloads compared as NaN==NaN). */
#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include "../../paper_2602_16760_b200/csrc/sfg_expf.h"

#define NT 16
static unsigned long long bad[NT];
static void* work(void* arg) {
    long t = (long)arg;
    uint64_t lo = ((uint64_t)1 << 32) / NT * t, hi = ((uint64_t)1 << 32) / NT * (t + 1);
    for (uint64_t u = lo; u < hi; ++u) {
        float x = sfg_as_f32_((uint32_t)u);
        float a = expf(x), b = sfg_expf(x);
        uint32_t ua = sfg_as_u32_(a), ub = sfg_as_u32_(b);
        if (ua != ub && !(isnan(a) && isnan(b))) {
            if (bad[t] < 3) fprintf(stderr, "x=%a libm=%a port=%a\n", x, a, b);
            bad[t]++;
        }
    }
    return NULL;
}
int main(void) {
    pthread_t th[NT];
    for (long t = 0; t < NT; ++t) pthread_create(&th[t], NULL, work, (void*)t);
    unsigned long long total = 0;
    for (int t = 0; t < NT; ++t) { pthread_join(th[t], NULL); total += bad[t]; }
    printf("mismatches %llu\n", total);
    return total != 0;
}

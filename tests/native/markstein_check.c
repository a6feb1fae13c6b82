/* Checks the division used by the GPU walk (siddon_walk.cuh div_rn):
 *   q0 = num * y,  r = fma(-q0, d, num),  q = fma(r, y, q0),  y = RN(1/d)
 * against IEEE-754 division over random operands spanning 2^-20..2^20 and
 * the geometry ranges the walk sees.  Prints the mismatch count. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
static uint64_t x = 88172645463325252ull;
static inline uint64_t rnd(void) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; return x; }
static inline double u01(void) { return (rnd() >> 11) * 0x1.0p-53; }
int main(int argc, char **argv) {
  long n = argc > 1 ? atol(argv[1]) : 20000000, bad = 0;
  for (long i = 0; i < n; i++) {
    double d, num;
    if (i & 1) {  /* geometry-like: plane coordinates minus sources over directions */
      d = (u01() - 0.5) * 2000.0;
      num = floor(u01() * 600.0) * 0.703125 - (u01() - 0.5) * 800.0;
    } else {
      d = (u01() - 0.5) * ldexp(1.0, (int)(rnd() % 40) - 20);
      num = (u01() - 0.5) * ldexp(1.0, (int)(rnd() % 40) - 20);
    }
    if (d == 0.0) continue;
    double y = 1.0 / d, q0 = num * y, r = fma(-q0, d, num), q = fma(r, y, q0);
    if (q != num / d) bad++;
  }
  printf("%ld\n", bad);
  return 0;
}

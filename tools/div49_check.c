/* Exhaustive check behind div49() in paper_2511_04261_b200/csrc/kernels.cu:
 * for every SSIM window sum x in [0, 49 * 255^2], RN(x * RN(1/49)) corrected
 * by one fma on the exact remainder equals the IEEE quotient x / 49.
 *   gcc -O2 -ffp-contract=off tools/div49_check.c -lm && ./a.out   -> bad=0 */
#include <math.h>
#include <stdio.h>
int main(void){
  const double r = 1.0/49.0; long bad=0;
  for (long x=0;x<=49L*65025L;++x){
    double a=(double)x, q=a*r, rem=fma(-q,49.0,a), q2=fma(rem,r,q);
    if (q2 != a/49.0){ if(bad<5) printf("bad %ld\n",x); ++bad; }
  }
  printf("bad=%ld\n",bad); return 0;}

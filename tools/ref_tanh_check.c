// ref_tanh_check.c -- host pin of the glibc tanh/expm1 restatement (tools/ref_tanh_host.h) that
// csrc/ref_tanh.cuh ports to the device:  gcc -O2 -ffp-contract=off tools/ref_tanh_check.c -lm
// && ./a.out 30000000   ->  "tanh mismatches 0, expm1 mismatches 0".
#include <stdio.h>
#include <stdlib.h>
#include "ref_tanh_host.h"
int main(int argc, char** argv){
  long N = argc>1 ? atol(argv[1]) : 50000000; long bad=0, bade=0; srand48(7);
  for(long i=0;i<N;i++){
    double mag = pow(10.0, drand48()*6.0-5.0);           /* 1e-5 .. 10 */
    double x = (drand48()<0.5?-1:1) * (i%4==0 ? drand48()*25.0 : mag);
    double a=tanh(x), bb=g_tanh(x);
    if(memcmp(&a,&bb,8)){ if(bad<5) printf("tanh x=%.17g libm=%.17g mine=%.17g\n",x,a,bb); bad++; }
    double y = (drand48()*2-1)*50.0; double c=expm1(y), d=g_expm1(y); if(memcmp(&c,&d,8)){ if(bade<5) printf("expm1 y=%.17g libm=%.17g mine=%.17g\n",y,c,d); bade++; }
  }
  double edge[]={0.0,-0.0,1e-300,-1e-300,5e-324,1e-17,0.5493061443340548,1.0,-1.0,21.999999,22.0,-22.0,1e300,INFINITY,-INFINITY,NAN,0.34657359027997264,1.0397207708399179};
  for(unsigned j=0;j<sizeof edge/sizeof*edge;j++){ double a=tanh(edge[j]), bb=g_tanh(edge[j]); if(memcmp(&a,&bb,8)){printf("edge %.17g libm=%.17g mine=%.17g\n",edge[j],a,bb); bad++;} }
  printf("tanh mismatches %ld, expm1 mismatches %ld of %ld\n", bad, bade, N);
  return bad!=0;
}

/* Restatement of this image's glibc 2.39 x86-64 tanh (baseline build) and the FMA
 * variant of expm1 it calls through the ifunc, from their machine code: fdlibm's
 * algorithm with an Estrin-form polynomial and the fused multiply-adds the compiler
 * emitted.  Every operation is explicit so the result is bit-identical.
 *
 * Derived from fdlibm (s_tanh.c, s_expm1.c) as shipped in glibc:
 *   Copyright (C) 1993 by Sun Microsystems, Inc. All rights reserved.
 *   Developed at SunPro, a Sun Microsystems, Inc. business.
 *   Permission to use, copy, modify, and distribute this software is freely granted,
 *   provided that this notice is preserved. */
#include <math.h>
#include <stdint.h>
#include <string.h>
static inline uint64_t g_bits(double x){uint64_t b; memcpy(&b,&x,8); return b;}
static inline double g_dbl(uint64_t b){double x; memcpy(&x,&b,8); return x;}
static inline double g_add_hi(double y, int32_t k){ /* high word += k << 20 */
  uint64_t b=g_bits(y); uint32_t hi=(uint32_t)(b>>32)+((uint32_t)k<<20); return g_dbl(((uint64_t)hi<<32)|(uint32_t)b); }
static double g_expm1(double x){
  const double invln2=1.4426950408889634, ln2_hi=0.6931471803691238, ln2_lo=1.9082149292705877e-10;
  const double Q1=-0.03333333333333313, Q2=0.0015873015872548146, Q3=-7.93650757867488e-05,
               Q4=4.008217827329362e-06, Q5=-2.0109921818362437e-07;
  uint64_t b=g_bits(x); uint32_t hx=(uint32_t)(b>>32)&0x7fffffffu; int neg=(int)(b>>63);
  double hi,lo,c=0.0; int32_t k;
  if(hx>0x40436879u){
    if(hx>0x40862e41u){
      if(hx>0x7fefffffu){ if((((uint32_t)(b>>32))&0xfffffu)|(uint32_t)b) return x+x; return neg?-1.0:x; }
      if(x>709.782712893384) return 1e300*1e300;
    }
    if(neg) return 1e-300-1.0;
    double t; k=(int32_t)(0.5+x*invln2); t=(double)k;
    hi=fma(-t,ln2_hi,x); lo=t*ln2_lo; x=hi-lo; c=(hi-x)-lo;
  } else if(hx>0x3fd62e42u){
    if(hx>0x3ff0a2b1u){
      double t; k=(int32_t)((neg?-0.5:0.5)+x*invln2); t=(double)k;
      hi=fma(-t,ln2_hi,x); lo=t*ln2_lo;
    } else if(!neg){ hi=x-ln2_hi; lo=ln2_lo; k=1; }
    else { hi=x+ln2_hi; lo=-ln2_lo; k=-1; }
    x=hi-lo; c=(hi-x)-lo;
  } else if(hx<=0x3c8fffffu){
    double t=x+1e300; t=t-t; return x-t;
  } else k=0;
  double hfx=x*0.5, hxs=x*hfx;
  double R2=fma(hxs,Q3,Q2), R3=fma(hxs,Q5,Q4), h2=hxs*hxs, R1=fma(hxs,Q1,1.0), h4=h2*h2;
  double r1=fma(h4,R3,fma(h2,R2,R1));
  double t=fma(-r1,hfx,3.0);
  double e=((r1-t)/fma(-x,t,6.0))*hxs;
  if(k==0) return x-fma(e,x,-hxs);
  e=fma(e-c,x,-c)-hxs;
  if(k==-1) return fma(x-e,0.5,-0.5);
  if(k==1){ if(x<-0.25) return (e-(x+0.5))*-2.0; return fma(x-e,2.0,1.0); }
  if((uint32_t)(k+1)>57u){ double y=1.0-(e-x); return g_add_hi(y,k)-1.0; }  /* k <= -2 or k > 56 */
  if(k<20){ double t2=g_dbl((uint64_t)(0x3ff00000u-(0x200000u>>k))<<32); return g_add_hi(t2-(e-x),k); }
  { double t2=g_dbl((uint64_t)((uint32_t)(0x3ff-k)<<20)<<32); double y=(x-(e+t2))+1.0; return g_add_hi(y,k); }
}
static double g_tanh(double x){
  uint64_t b=g_bits(x); uint32_t jx=(uint32_t)(b>>32), ix=jx&0x7fffffffu; double z;
  if(ix>0x7fefffffu) return (int32_t)jx>=0 ? 1.0/x+1.0 : 1.0/x-1.0;
  if(ix<=0x4035ffffu){
    if((ix|(uint32_t)b)==0) return x;
    double ax=fabs(x);
    if(ix<=0x3c7fffffu) return (1.0+x)*x;
    if(ix<=0x3fefffffu){ double t=g_expm1(ax*-2.0); z=(-t)/(t+2.0); }
    else { double t=g_expm1(ax+ax); z=1.0-2.0/(t+2.0); }
  } else z=1.0-1e-300;
  return (int32_t)jx>=0 ? z : -z;
}

/* Branch-free form of g_tanh for the device: the same operations, every reconstruction
 * computed and selected (lanes of a warp take different expm1 branches otherwise). */
static double g_tanh_bf(double x){
  const double invln2=1.4426950408889634, ln2_hi=0.6931471803691238, ln2_lo=1.9082149292705877e-10;
  const double Q1=-0.03333333333333313, Q2=0.0015873015872548146, Q3=-7.93650757867488e-05,
               Q4=4.008217827329362e-06, Q5=-2.0109921818362437e-07;
  uint64_t b=g_bits(x); uint32_t ix=(uint32_t)(b>>32)&0x7fffffffu;
  double ax=fabs(x); int small = ix<=0x3fefffffu;                   /* |x| < 1 */
  double a = small ? ax*-2.0 : ax+ax;                               /* expm1 argument */
  uint32_t ha=(uint32_t)(g_bits(a)>>32)&0x7fffffffu;
  int k = ha<=0x3fd62e42u ? 0 : (int32_t)((a<0?-0.5:0.5)+a*invln2);
  double tk=(double)k, hi=fma(-tk,ln2_hi,a), lo=tk*ln2_lo, xr=hi-lo, c=(hi-xr)-lo;
  double hfx=xr*0.5, hxs=xr*hfx;
  double R2=fma(hxs,Q3,Q2), R3=fma(hxs,Q5,Q4), h2=hxs*hxs, R1=fma(hxs,Q1,1.0), h4=h2*h2;
  double r1=fma(h4,R3,fma(h2,R2,R1)), t=fma(-r1,hfx,3.0);
  double e=((r1-t)/fma(-xr,t,6.0))*hxs;
  double r0=xr-fma(e,xr,-hxs);
  double e2=fma(e-c,xr,-c)-hxs;
  double rm1=fma(xr-e2,0.5,-0.5);
  double rp1= xr<-0.25 ? (e2-(xr+0.5))*-2.0 : fma(xr-e2,2.0,1.0);
  double rbig=g_add_hi(1.0-(e2-xr),k)-1.0;
  int kl = k<0?0:(k>19?19:k);
  double rmid=g_add_hi(g_dbl((uint64_t)(0x3ff00000u-(0x200000u>>kl))<<32)-(e2-xr),k);
  int kh = k<20?20:(k>1023?1023:k);
  double rhi=g_add_hi((xr-(e2+g_dbl((uint64_t)((uint32_t)(0x3ff-kh)<<20)<<32)))+1.0,k);
  double em1 = k==0 ? r0 : k==-1 ? rm1 : k==1 ? rp1 : ((uint32_t)(k+1)>57u ? rbig : (k<20 ? rmid : rhi));
  double q=(small ? -em1 : 2.0)/(em1+2.0);
  double z = small ? q : 1.0-q;
  if(ix>0x4035ffffu) z=1.0;                                          /* |x| >= 22 */
  if(ix<=0x3c7fffffu) return (ix|(uint32_t)b)==0 ? x : (1.0+x)*x;    /* |x| < 2^-55, +-0 */
  return (int64_t)b>=0 ? z : -z;
}

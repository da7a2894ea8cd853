/* Restatement of glibc 2.39 tanh/expm1 (fdlibm s_tanh.c, s_expm1.c) checked
 * against the host libm: build with  gcc -O2 -mfma -ffp-contract=fast
 * tanh_glibc.c -lm  (FMA ifunc build of expm1, Estrin polynomial: 0
 * mismatches) and with -ffp-contract=off (non-FMA build). The device copy is
 * csrc/cuda/libm_glibc.cuh; contraction sites read off -fdump-tree-widening_mul. */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
static inline uint32_t HI(double x){uint64_t u;memcpy(&u,&x,8);return u>>32;}
static inline uint32_t LO(double x){uint64_t u;memcpy(&u,&x,8);return (uint32_t)u;}
static inline double SETHI(double x, uint32_t h){uint64_t u;memcpy(&u,&x,8);u=(u&0xffffffffull)|((uint64_t)h<<32);memcpy(&x,&u,8);return x;}
static const double one=1.0,huge=1.0e+300,tiny=1.0e-300,o_threshold=7.09782712893383973096e+02,
ln2_hi=6.93147180369123816490e-01,ln2_lo=1.90821492927058770002e-10,invln2=1.44269504088896338700e+00,
Q1=-3.33333333333331316428e-02,Q2=1.58730158725481460165e-03,Q3=-7.93650757867487942473e-05,
Q4=4.00821782732936239552e-06,Q5=-2.01099218183624371326e-07;
double my_expm1(double x, int estrin){
  double y,hi,lo,c=0,t,e,hxs,hfx,r1; int k,xsb; uint32_t hx;
  hx=HI(x); xsb=hx&0x80000000; y= xsb==0?x:-x; hx&=0x7fffffff;
  if(hx>=0x4043687A){ if(hx>=0x40862E42){ if(hx>=0x7ff00000){ if(((hx&0xfffff)|LO(x))!=0) return x+x; else return xsb==0?x:-1.0;} if(x>o_threshold) return huge*huge;}
    if(xsb!=0){ if(x+tiny<0.0) return tiny-one;}}
  if(hx>0x3fd62e42){ if(hx<0x3FF0A2B2){ if(xsb==0){hi=x-ln2_hi;lo=ln2_lo;k=1;} else {hi=x+ln2_hi;lo=-ln2_lo;k=-1;} }
    else { k=invln2*x+((xsb==0)?0.5:-0.5); t=k; hi=x-t*ln2_hi; lo=t*ln2_lo; }
    x=hi-lo; c=(hi-x)-lo; }
  else if(hx<0x3c900000){ t=huge+x; return x-(t-(huge+x)); }
  else k=0;
  hfx=0.5*x; hxs=x*hfx;
  if(estrin){ double R1=one+hxs*Q1, h2=hxs*hxs, R2=Q2+hxs*Q3, h4=h2*h2, R3=Q4+hxs*Q5; r1=R1+h2*R2+h4*R3; }
  else r1=one+hxs*(Q1+hxs*(Q2+hxs*(Q3+hxs*(Q4+hxs*Q5))));
  t=3.0-r1*hfx; e=hxs*((r1-t)/(6.0-x*t));
  if(k==0) return x-(x*e-hxs);
  e=(x*(e-c)-c); e-=hxs;
  if(k==-1) return 0.5*(x-e)-0.5;
  if(k==1){ if(x<-0.25) return -2.0*(e-(x+0.5)); else return one+2.0*(x-e); }
  if(k<=-2||k>56){ y=one-(e-x); y=SETHI(y,HI(y)+(k<<20)); return y-one; }
  t=one;
  if(k<20){ t=SETHI(t,0x3ff00000-(0x200000>>k)); y=t-(e-x); y=SETHI(y,HI(y)+(k<<20)); }
  else { t=SETHI(t,((0x3ff-k)<<20)); y=x-(e+t); y+=one; y=SETHI(y,HI(y)+(k<<20)); }
  return y;
}
double my_tanh(double x, int estrin){
  double t,z; int32_t jx=(int32_t)HI(x), ix=jx&0x7fffffff; uint32_t lx=LO(x);
  if(ix>=0x7ff00000){ if(jx>=0) return one/x+one; else return one/x-one; }
  if(ix<0x40360000){ if((ix|lx)==0) return x; if(ix<0x3c800000) return x*(one+x);
    if(ix>=0x3ff00000){ t=my_expm1(2.0*fabs(x),estrin); z=one-2.0/(t+2.0);} else { t=my_expm1(-2.0*fabs(x),estrin); z=-t/(t+2.0);} }
  else z=one-tiny;
  return jx>=0?z:-z;
}
int main(){
  uint64_t s=88172645463325252ull; long bad[2]={0,0}, badx[2]={0,0}; long N=20000000;
  for(long i=0;i<N;i++){ s^=s<<13;s^=s>>7;s^=s<<17;
    double u=(double)(s>>11)/9007199254740992.0; double x = (i&1?-1:1)*exp(-20+ 24*u); /* |x| in e^-20..e^4 */
    double g=tanh(x);
    for(int v=0;v<2;v++){ double m=my_tanh(x,v); if(m!=g) bad[v]++; double ge=expm1(x), me=my_expm1(x,v); if(ge!=me) badx[v]++; }
  }
  printf("tanh mismatches horner=%ld estrin=%ld ; expm1 mismatches horner=%ld estrin=%ld of %ld\n",bad[0],bad[1],badx[0],badx[1],N);
}

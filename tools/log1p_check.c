// Host check (tools only): the restated glibc log1p (FMA build) vs the C library
// log1p, bitwise; build: gcc -O2 -ffp-contract=off -o /tmp/l1p tools/log1p_check.c -lm
#include <math.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>
#include <stdlib.h>
static const double ln2_hi=6.93147180369123816490e-01, ln2_lo=1.90821492927058770002e-10, two54=1.80143985094819840000e+16,
Lp1=6.666666666666735130e-01,Lp2=3.999999999940941908e-01,Lp3=2.857142874366239149e-01,Lp4=2.222219843214978396e-01,
Lp5=1.818357216161805012e-01,Lp6=1.531383769920937332e-01,Lp7=1.479819860511658591e-01;
static inline int32_t hiw(double x){uint64_t u;memcpy(&u,&x,8);return (int32_t)(u>>32);}
static inline double sethi(double x,int32_t h){uint64_t u;memcpy(&u,&x,8);u=(u&0xffffffffull)|((uint64_t)(uint32_t)h<<32);memcpy(&x,&u,8);return x;}
double ex_log1p(double x){
  double hfsq,f=0,c=0,s,z,R,u;
  int32_t k,hx,hu=0,ax;
  hx=hiw(x); ax=hx&0x7fffffff; k=1;
  if(hx<0x3FDA827A){
    if(ax>=0x3ff00000){ if(x==-1.0) return -two54/0.0; else return (x-x)/(x-x);}
    if(ax<0x3e200000){ if(two54+x>0.0 && ax<0x3c900000) return x; else return fma(-(x*x),0.5,x);}
    if(hx>0||hx<=((int32_t)0xbfd2bec3)){k=0;f=x;hu=1;}
  }
  if(hx>=0x7ff00000) return x+x;
  if(k!=0){
    if(hx<0x43400000){ u=1.0+x; hu=hiw(u); k=(hu>>20)-1023; c=(k>0)?1.0-(u-x):x-(u-1.0); c/=u; }
    else { u=x; hu=hiw(u); k=(hu>>20)-1023; c=0; }
    hu&=0x000fffff;
    if(hu<0x6a09e){ u=sethi(u,hu|0x3ff00000);} else { k+=1; u=sethi(u,hu|0x3fe00000); hu=(0x00100000-hu)>>2; }
    f=u-1.0;
  }
  hfsq=(0.5*f)*f;
  const double dk=(double)k;
  if(hu==0){
    if(f==0.0){ if(k==0) return 0.0; else {c=fma(dk,ln2_lo,c); return fma(dk,ln2_hi,c);} }
    R=fma(-f,0.66666666666666666,1.0)*hfsq;
    if(k==0) return f-R; else return fma(dk,ln2_hi,-((R-fma(dk,ln2_lo,c))-f));
  }
  s=f/(2.0+f);
  z=s*s;
  double R2=fma(Lp3,z,Lp2), R3=fma(Lp5,z,Lp4), R4=fma(Lp7,z,Lp6);
  double z2=z*z, z4=z2*z2, z6=z4*z2;
  R=fma(z,Lp1,z2*R2); R=fma(z4,R3,R); R=fma(z6,R4,R);
  double t=s*(R+hfsq);
  if(k==0) return f-(hfsq-t);
  return fma(dk,ln2_hi,-((hfsq-(fma(dk,ln2_lo,c)+t))-f));
}
int main(int argc,char**argv){
  long N=atol(argv[1]); uint64_t st=88172645463325252ull; long bad=0;
  for(long i=0;i<N;i++){
    st^=st<<13; st^=st>>7; st^=st<<17;
    double u;
    if(i%4==0) u=(double)(st>>11)*(1.0/9007199254740992.0);
    else if(i%4==1) u=ldexp((double)(st>>11)*(1.0/9007199254740992.0), -(int)(st%60));  // small |x|
    else if(i%4==2) {uint64_t b=st>>1; double v; memcpy(&v,&b,8); if(!(v==v)||isinf(v)) continue; u=-v;} // any double
    else u=1.0-(double)(st>>11)*(1.0/9007199254740992.0)*1e-3;
    double a=log1p(-u), b=ex_log1p(-u);
    if(memcmp(&a,&b,8) && !(a!=a && b!=b)){ if(bad<5) printf("%.17g %.17g %.17g\n",u,a,b); bad++;}
  }
  printf("N=%ld bad=%ld\n",N,bad);
}

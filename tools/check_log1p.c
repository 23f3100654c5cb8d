#include <math.h>
#include <stdio.h>
#include <stdint.h>
#include <string.h>
static int hiw(double x){uint64_t b; memcpy(&b,&x,8); return (int)(b>>32);}
static double sethi(double x, uint32_t h){uint64_t b; memcpy(&b,&x,8); b=(b&0xffffffffULL)|((uint64_t)h<<32); memcpy(&x,&b,8); return x;}
static const double ln2_hi=6.93147180369123816490e-01, ln2_lo=1.90821492927058770002e-10,
Lp1=6.666666666666735130e-01,Lp2=3.999999999940941908e-01,Lp3=2.857142874366239149e-01,Lp4=2.222219843214978396e-01,
Lp5=1.818357216161805012e-01,Lp6=1.531383769920937332e-01,Lp7=1.479819860511658591e-01;
/* restatement of glibc 2.39 __log1p_fma (x86-64 FMA multiarch), for x in (-1, 0.41) */
double my_log1p(double x){
  double hfsq,f,c=0,s,z,R,u; int k,hx,hu=0,ax;
  hx=hiw(x); ax=hx&0x7fffffff; k=1;
  if(hx<0x3FDA827A){
    if(ax>=0x3ff00000){ return x==-1.0 ? -INFINITY : NAN;}
    if(ax<0x3e200000){ if(ax<0x3c900000) return x; return fma(-(x*x),0.5,x);}
    if(hx>0||hx<=((int)0xbfd2bec3)){k=0;f=x;hu=1;}
  }
  if(k!=0){
    u=1.0+x; hu=hiw(u); k=(hu>>20)-1023; c=(k>0)?1.0-(u-x):x-(u-1.0); c/=u;
    hu&=0x000fffff;
    if(hu<0x6a09e){ u=sethi(u,hu|0x3ff00000);} else {k+=1; u=sethi(u,hu|0x3fe00000); hu=(0x00100000-hu)>>2;}
    f=u-1.0;
  }
  hfsq=(0.5*f)*f;
  if(hu==0){
    if(f==0.0){ if(k==0) return 0.0; double kd=k; return fma(kd,ln2_hi,fma(kd,ln2_lo,c));}
    R=fma(-f,0.6666666666666666,1.0)*hfsq;
    if(k==0) return f-R; double kd=k; return fma(kd,ln2_hi,-((R-fma(kd,ln2_lo,c))-f));
  }
  s=f/(2.0+f); z=s*s;
  { double Ra=fma(z,Lp3,Lp2), Rb=fma(z,Lp5,Lp4), Rc=fma(z,Lp7,Lp6), z2=z*z, z4=z2*z2, z6=z2*z4;
    R=fma(z6,Rc,fma(z4,Rb,fma(z,Lp1,z2*Ra))); }
  double t=s*(R+hfsq);
  if(k==0) return f-(hfsq-t);
  double kd=k; double q=fma(kd,ln2_lo,c)+t; q=(hfsq-q)-f; return fma(kd,ln2_hi,-q);
}
int main(){
  uint64_t st=88172645463325252ULL; long bad=0, n=400000000;
  for(long i=0;i<n;i++){ st^=st<<13; st^=st>>7; st^=st<<17;
    double u=(double)(st>>11)*(1.0/9007199254740992.0);
    double x = (i%3==0)? -u : (i%3==1 ? -u*ldexp(1.0,-(int)(i%60)) : -u*1e-3*(double)(i%7));
    double a=log1p(x), b=my_log1p(x);
    if(memcmp(&a,&b,8)){ if(bad<5) printf("x=%.17g glibc=%.17g mine=%.17g\n",x,a,b); bad++;}
  }
  printf("mismatches %ld / %ld\n",bad,n);
}

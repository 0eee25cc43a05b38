#define _POSIX_C_SOURCE 199309L
#include "egs_oracle.h"
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
static double now(void){struct timespec ts;clock_gettime(CLOCK_MONOTONIC,&ts);return ts.tv_sec+ts.tv_nsec*1e-9;}
/* certificate: returns number of vertices newly set to TOP */
static const int64_t* g_prev=0;
static uint64_t certify(const eo_arena*g,int64_t*f,uint8_t*cand,int64_t*snap,int*passes){
  uint32_t n=g->n; memcpy(snap,f,n*8); if(getenv("JSTEP")) for(uint32_t v=0;v<n;v++){int64_t c=eo_raw_lift(g,v,f); if(c>snap[v]) snap[v]=c;}
  for(uint32_t v=0;v<n;v++) cand[v]=snap[v]!=EO_TOP && (!getenv("CANDCHG") || !g_prev || g_prev[v]!=f[v]);
  uint64_t nc=0; for(uint32_t v=0;v<n;v++) nc+=cand[v]; if(getenv("VERB")) fprintf(stderr,"  cand=%llu\n",(unsigned long long)nc);
  int changed=1; *passes=0;
  while(changed){changed=0;(*passes)++;
    for(uint32_t v=0;v<n;v++){ if(!cand[v]) continue; int ok;
      if(g->owner[v]==0){ ok=1; for(uint64_t i=g->csr_off[v];i<g->csr_off[v+1];i++){uint32_t t=g->csr_dst[i]; int64_t w=g->csr_w[i];
          if(snap[t]==EO_TOP) continue; if(!(cand[t] && snap[v] < snap[t]-w)){ok=0;break;}}}
      else { ok=0; for(uint64_t i=g->csr_off[v];i<g->csr_off[v+1];i++){uint32_t t=g->csr_dst[i]; int64_t w=g->csr_w[i];
          if(snap[t]==EO_TOP || (cand[t] && snap[v] < snap[t]-w)){ok=1;break;}}}
      if(!ok){cand[v]=0;changed=1;}
    }}
  uint64_t c=0; for(uint32_t v=0;v<n;v++) if(cand[v]){f[v]=EO_TOP;c++;}
  return c;
}
int main(int argc,char**argv){
  eo_arena g; int rc;
  if(!strcmp(argv[1],"fixed")) rc=eo_gen_fixed(atoll(argv[2]),atoi(argv[3]),atoll(argv[4]),1,&g);
  else rc=eo_gen_rmat(atoi(argv[2]),atoi(argv[3]),atoll(argv[4]),1,&g);
  if(rc) return 1;
  int jacobi=atoi(argv[5]); int K=atoi(argv[6]);
  uint32_t n=g.n; int64_t*ref=calloc(n,8); eo_stats st; if(!getenv("NOREF")) eo_solve_seq(&g,ref,&st);
  int64_t*f=calloc(n,8),*prev=malloc(n*8),*snap=malloc(n*8); uint8_t*cand=malloc(n);
  uint64_t rounds=0, certs=0, ncert=0, totpass=0; double t0=now();
  for(;;){ int changed=0; if(jacobi) memcpy(prev,f,n*8);
    const int64_t* src = jacobi?prev:f;
    for(uint32_t v=0;v<n;v++){ int64_t c=eo_raw_lift(&g,v,src); if(c>f[v]){f[v]=c;changed=1;} }
    rounds++;
    if(!changed) break; if(rounds%1000==0) fprintf(stderr,"r%llu\n",(unsigned long long)rounds); if(getenv("MAXR") && rounds>=atoll(getenv("MAXR"))) break;
    if(K>0 && rounds%K==0){int p; g_prev=jacobi?prev:0; uint64_t c=certify(&g,f,cand,snap,&p); certs++; ncert+=c; totpass+=p;
       if(c) fprintf(stderr,"  round %llu: certified %llu (passes %d)\n",(unsigned long long)rounds,(unsigned long long)c,p);}
  }
  uint64_t tops=0; long long sum=0; int64_t mx=0; for(uint32_t v=0;v<n;v++){ if(f[v]==EO_TOP) tops++; else {sum+=f[v]; if(f[v]>mx) mx=f[v];}} fprintf(stderr,"tops=%llu sum=%lld max=%lld pm=%d\n",(unsigned long long)tops,sum,(long long)mx,eo_is_progress_measure(&g,f));
  uint64_t mis=0; for(uint32_t v=0;v<n;v++) if(f[v]!=ref[v]) mis++;
  printf("%s %s %s %s jacobi=%d K=%d rounds=%llu certs=%llu certified=%llu passes=%llu mismatches=%llu time=%.2f\n",argv[1],argv[2],argv[3],argv[4],jacobi,K,
    (unsigned long long)rounds,(unsigned long long)certs,(unsigned long long)ncert,(unsigned long long)totpass,(unsigned long long)mis,now()-t0);
}

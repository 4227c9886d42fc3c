// Instruction-throughput microbenchmarks for sm_100a (dev tool). Each kernel runs
// NW warps per CTA x (SMs*k) CTAs; each thread executes ITERS x 8 independent ops.
// Reports warp-instructions per SM per clock.
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#define ITERS 1024
__device__ uint32_t sink;
#define BODY8(OP) OP(0) OP(1) OP(2) OP(3) OP(4) OP(5) OP(6) OP(7)

template<int K> __global__ void k_popc(uint32_t seed, long long* cyc) {
  uint32_t r[8]; for (int i=0;i<8;++i) r[i] = seed*(threadIdx.x+i+1);
  long long t0 = clock64();
  for (int it=0; it<ITERS; ++it) {
#define OP(i) r[i] = __popc(r[i]) ^ r[(i+1)&7];
    BODY8(OP)
#undef OP
  }
  long long t1 = clock64();
  uint32_t s=0; for (int i=0;i<8;++i) s+=r[i]; if (s==12345) sink=s;
  if (threadIdx.x==0) cyc[blockIdx.x]=t1-t0;
}
template<int K> __global__ void k_flo(uint32_t seed, long long* cyc) {
  uint32_t r[8]; for (int i=0;i<8;++i) r[i] = seed*(threadIdx.x+i+1);
  long long t0 = clock64();
  for (int it=0; it<ITERS; ++it) {
#define OP(i) r[i] = __clz(r[i]) ^ r[(i+1)&7];
    BODY8(OP)
#undef OP
  }
  long long t1 = clock64();
  uint32_t s=0; for (int i=0;i<8;++i) s+=r[i]; if (s==12345) sink=s;
  if (threadIdx.x==0) cyc[blockIdx.x]=t1-t0;
}
template<int K> __global__ void k_prmt(uint32_t seed, long long* cyc) {
  uint32_t r[8]; for (int i=0;i<8;++i) r[i] = seed*(threadIdx.x+i+1);
  uint32_t sel = seed ^ threadIdx.x;
  long long t0 = clock64();
  for (int it=0; it<ITERS; ++it) {
#define OP(i) r[i] = __byte_perm(r[i], r[(i+3)&7], sel + i);
    BODY8(OP)
#undef OP
  }
  long long t1 = clock64();
  uint32_t s=0; for (int i=0;i<8;++i) s+=r[i]; if (s==12345) sink=s;
  if (threadIdx.x==0) cyc[blockIdx.x]=t1-t0;
}
template<int K> __global__ void k_lop(uint32_t seed, long long* cyc) {
  uint32_t r[8]; for (int i=0;i<8;++i) r[i] = seed*(threadIdx.x+i+1);
  long long t0 = clock64();
  for (int it=0; it<ITERS; ++it) {
#define OP(i) r[i] = (r[i] & r[(i+3)&7]) ^ r[(i+5)&7];
    BODY8(OP)
#undef OP
  }
  long long t1 = clock64();
  uint32_t s=0; for (int i=0;i<8;++i) s+=r[i]; if (s==12345) sink=s;
  if (threadIdx.x==0) cyc[blockIdx.x]=t1-t0;
}
template<int K> __global__ void k_imad(uint32_t seed, long long* cyc) {
  uint32_t r[8]; for (int i=0;i<8;++i) r[i] = seed*(threadIdx.x+i+1);
  long long t0 = clock64();
  for (int it=0; it<ITERS; ++it) {
#define OP(i) r[i] = r[i] * r[(i+3)&7] + r[(i+5)&7];
    BODY8(OP)
#undef OP
  }
  long long t1 = clock64();
  uint32_t s=0; for (int i=0;i<8;++i) s+=r[i]; if (s==12345) sink=s;
  if (threadIdx.x==0) cyc[blockIdx.x]=t1-t0;
}
template<int K> __global__ void k_shfl(uint32_t seed, long long* cyc) {
  uint32_t r[8]; for (int i=0;i<8;++i) r[i] = seed*(threadIdx.x+i+1);
  long long t0 = clock64();
  for (int it=0; it<ITERS; ++it) {
#define OP(i) r[i] = __shfl_sync(0xffffffffu, r[i], r[(i+1)&7]);
    BODY8(OP)
#undef OP
  }
  long long t1 = clock64();
  uint32_t s=0; for (int i=0;i<8;++i) s+=r[i]; if (s==12345) sink=s;
  if (threadIdx.x==0) cyc[blockIdx.x]=t1-t0;
}
// shared loads: per-lane addresses conflict-free
template<int W> __global__ void k_lds(uint32_t seed, long long* cyc) {
  __shared__ __align__(16) uint32_t sm[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i * seed;
  __syncthreads();
  uint32_t r[8]; for (int i=0;i<8;++i) r[i] = (threadIdx.x & 31) * W + i;
  long long t0 = clock64();
  for (int it=0; it<ITERS; ++it) {
    if (W == 1) {
#define OP(i) r[i] = sm[(r[i] & 1023) ];
      BODY8(OP)
#undef OP
    } else if (W == 2) {
#define OP(i) { uint2 v = reinterpret_cast<const uint2*>(sm)[(r[i] & 1023)]; r[i] = v.x ^ v.y; }
      BODY8(OP)
#undef OP
    } else if (W == 4) {
#define OP(i) { uint4 v = reinterpret_cast<const uint4*>(sm)[(r[i] & 1023)]; r[i] = v.x ^ v.w; }
      BODY8(OP)
#undef OP
    } else {  // u16
#define OP(i) r[i] = reinterpret_cast<const uint16_t*>(sm)[(r[i] & 2047)];
      BODY8(OP)
#undef OP
    }
  }
  long long t1 = clock64();
  uint32_t s=0; for (int i=0;i<8;++i) s+=r[i]; if (s==12345) sink=s;
  if (threadIdx.x==0) cyc[blockIdx.x]=t1-t0;
}
template<int K> __global__ void k_hmma(uint32_t seed, long long* cyc) {
  float d[4][4] = {}; uint32_t a = seed ^ threadIdx.x, b = seed * 3;
  long long t0 = clock64();
  for (int it=0; it<ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%4,%4,%4}, {%5,%5}, {%0,%1,%2,%3};"
        : "+f"(d[i][0]), "+f"(d[i][1]), "+f"(d[i][2]), "+f"(d[i][3]) : "r"(a), "r"(b));
  }
  long long t1 = clock64();
  float s = 0; for (int i=0;i<4;++i) s += d[i][0]+d[i][1]+d[i][2]+d[i][3]; if (s==1.2345f) sink=1;
  if (threadIdx.x==0) cyc[blockIdx.x]=t1-t0;
}
template<int K> __global__ void k_movm(uint32_t seed, long long* cyc) {
  uint32_t r[8]; for (int i=0;i<8;++i) r[i] = seed*(threadIdx.x+i+1);
  long long t0 = clock64();
  for (int it=0; it<ITERS; ++it) {
#define OP(i) asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %0;" : "+r"(r[i]));
    BODY8(OP)
#undef OP
  }
  long long t1 = clock64();
  uint32_t s=0; for (int i=0;i<8;++i) s+=r[i]; if (s==12345) sink=s;
  if (threadIdx.x==0) cyc[blockIdx.x]=t1-t0;
}
template<int K> __global__ void k_fhfma(uint32_t seed, long long* cyc) {
  float f[8]; for (int i=0;i<8;++i) f[i] = seed*(threadIdx.x+i+1)*1e-9f;
  unsigned short h = seed & 0x3fff, h2 = (seed >> 3) & 0x3fff;
  long long t0 = clock64();
  for (int it=0; it<ITERS; ++it) {
#define OP(i) asm volatile("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(f[i]) : "h"(h), "h"(h2));
    BODY8(OP)
#undef OP
  }
  long long t1 = clock64();
  float s=0; for (int i=0;i<8;++i) s+=f[i]; if (s==1.2345f) sink=1;
  if (threadIdx.x==0) cyc[blockIdx.x]=t1-t0;
}

template <typename F>
void run(const char* name, F kern, int ops_per_iter, int nthreads) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* cyc; cudaMalloc(&cyc, sizeof(long long) * sms * 2);
  int blocks = sms * 2;
  kern<<<blocks, nthreads>>>(7u, cyc);
  cudaDeviceSynchronize();
  kern<<<blocks, nthreads>>>(7u, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[1024]; cudaMemcpy(h, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < blocks; ++i) avg += h[i]; avg /= blocks;
  // 2 CTAs per SM assumed co-resident
  double warp_instr = (double)ITERS * ops_per_iter * (nthreads / 32) * 2;
  printf("%-8s %s: %.3f warp-instr/clk/SM  (%.1f lanes/clk/SM)\n", name, e==cudaSuccess?"ok":cudaGetErrorString(e),
         warp_instr / avg, 32 * warp_instr / avg);
  cudaFree(cyc);
}

int main() {
  run("POPC", k_popc<0>, 8, 512);
  run("FLO", k_flo<0>, 8, 512);
  run("PRMT", k_prmt<0>, 8, 512);
  run("LOP3", k_lop<0>, 8, 512);
  run("IMAD", k_imad<0>, 8, 512);
  run("SHFL", k_shfl<0>, 8, 512);
  run("LDS.U16", k_lds<0>, 8, 512);
  run("LDS.32", k_lds<1>, 8, 512);
  run("LDS.64", k_lds<2>, 8, 512);
  run("LDS.128", k_lds<4>, 8, 512);
  run("HMMA", k_hmma<0>, 4, 512);
  run("MOVM", k_movm<0>, 8, 512);
  run("FHFMA", k_fhfma<0>, 8, 512);
  return 0;
}

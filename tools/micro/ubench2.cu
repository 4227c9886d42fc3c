// BMMA (b1 and.popc) / IMMA throughput + fragment layout probe (dev tool)
#include <cstdio>
#include <cstdint>
#include <algorithm>
#define ITERS 1024
__device__ uint32_t sink;
__global__ void k_bmma(uint32_t seed, long long* cyc) {
  int d[4][4] = {}; uint32_t a = seed ^ threadIdx.x, b = seed * 3;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%4,%4,%4}, {%5,%5}, {%0,%1,%2,%3};"
        : "+r"(d[i][0]), "+r"(d[i][1]), "+r"(d[i][2]), "+r"(d[i][3]) : "r"(a), "r"(b));
  }
  long long t1 = clock64();
  int s = 0; for (int i=0;i<4;++i) s += d[i][0]+d[i][1]+d[i][2]+d[i][3]; if (s==12345) sink=s;
  if (threadIdx.x==0) cyc[blockIdx.x]=t1-t0;
}
__global__ void k_imma(uint32_t seed, long long* cyc) {
  int d[4][4] = {}; uint32_t a = seed ^ threadIdx.x, b = seed * 3;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%4,%4,%4}, {%5,%5}, {%0,%1,%2,%3};"
        : "+r"(d[i][0]), "+r"(d[i][1]), "+r"(d[i][2]), "+r"(d[i][3]) : "r"(a), "r"(b));
  }
  long long t1 = clock64();
  int s = 0; for (int i=0;i<4;++i) s += d[i][0]+d[i][1]+d[i][2]+d[i][3]; if (s==12345) sink=s;
  if (threadIdx.x==0) cyc[blockIdx.x]=t1-t0;
}
// random-ish gather LDS.32 with realistic pattern: 8 tokens x 4 lanes, index = 41*g + 10*t + rand(0..9)
template <int stride> __global__ void k_gather(uint32_t seed, long long* cyc) {
  __shared__ uint32_t sm[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i;
  __syncthreads();
  int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  uint32_t x = seed * 2654435761u ^ threadIdx.x * 97u;
  uint32_t acc = 0;
  int base = (threadIdx.x >> 5) * 1024 + stride * g + 10 * t;
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      x = x * 1664525u + 1013904223u;
      acc += sm[(base + (x >> 28) % 10 + (acc & 0)) & 8191];
    }
  }
  long long t1 = clock64();
  if (acc == 12345) sink = acc;
  if (threadIdx.x==0) cyc[blockIdx.x]=t1-t0;
}
// layout probe: A row r has bits = r (in low bits of k), B col n has all bits set in k<64
__global__ void probe(int* out) {
  int lane = threadIdx.x;
  int g = lane >> 2, t = lane & 3;
  // A fragment guess: a0 = row g, k bits [32t, 32t+32); a1 = row g+8 ...; a2 = row g, k [128+32t..); a3 = row g+8
  // encode: row r's k-bits: set bit k iff k < (r+1) * 8  (so popc with all-ones col = 8(r+1) within k<128)
  auto rowbits = [](int r, int kbase) -> uint32_t { uint32_t v = 0; for (int i = 0; i < 32; ++i) if (kbase + i < (r + 1) * 8) v |= 1u << i; return v; };
  uint32_t a0 = rowbits(g, 32 * t), a1 = rowbits(g + 8, 32 * t), a2 = 0, a3 = 0;
  // B: col n has bits k < 16*(n+1)  (guess b0 = col g, k [32t..32t+32), b1 = col g, k [128+32t..])
  auto colbits = [](int n, int kbase) -> uint32_t { uint32_t v = 0; for (int i = 0; i < 32; ++i) if (kbase + i < 16 * (n + 1)) v |= 1u << i; return v; };
  uint32_t b0 = colbits(g, 32 * t), b1 = 0;
  int d0 = 0, d1 = 0, d2 = 0, d3 = 0;
  asm volatile("mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
    : "+r"(d0), "+r"(d1), "+r"(d2), "+r"(d3) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  out[lane * 4 + 0] = d0; out[lane * 4 + 1] = d1; out[lane * 4 + 2] = d2; out[lane * 4 + 3] = d3;
}
template <typename F> void run(const char* name, F kern, int ops, int nthreads) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* cyc; cudaMalloc(&cyc, sizeof(long long) * sms * 2);
  int blocks = sms * 2;
  kern<<<blocks, nthreads>>>(7u, cyc); cudaDeviceSynchronize();
  kern<<<blocks, nthreads>>>(7u, cyc); cudaError_t e = cudaDeviceSynchronize();
  long long h[1024]; cudaMemcpy(h, cyc, sizeof(long long) * blocks, cudaMemcpyDeviceToHost);
  double avg = 0; for (int i = 0; i < blocks; ++i) avg += h[i]; avg /= blocks;
  double wi = (double)ITERS * ops * (nthreads / 32) * 2;
  printf("%-10s %s: %.3f warp-instr/clk/SM\n", name, e == cudaSuccess ? "ok" : cudaGetErrorString(e), wi / avg);
}
int main() {
  run("BMMA", k_bmma, 4, 512);
  run("IMMA", k_imma, 4, 512);
  run("GATHER32", k_gather<32>, 8, 512);
  run("GATHER40", k_gather<40>, 8, 512);
  run("GATHER41", k_gather<41>, 8, 512);
  run("GATHER44", k_gather<44>, 8, 512);
  int* d; cudaMalloc(&d, 512); probe<<<1, 32>>>(d); int h[128]; cudaMemcpy(h, d, 512, cudaMemcpyDeviceToHost);
  printf("probe (expect D[r][n] = min(8(r+1),16(n+1)) if layout guess right)\n");
  for (int l = 0; l < 32; ++l) {
    int g = l >> 2, t = l & 3;
    int e0 = std::min(8 * (g + 1), 16 * (2 * t + 1)), e1 = std::min(8 * (g + 1), 16 * (2 * t + 2));
    int e2 = std::min(8 * (g + 9), 16 * (2 * t + 1)), e3 = std::min(8 * (g + 9), 16 * (2 * t + 2));
    printf("lane %2d: %3d %3d %3d %3d   expect %3d %3d %3d %3d %s\n", l, h[4*l], h[4*l+1], h[4*l+2], h[4*l+3], e0, e1, e2, e3,
           (h[4*l]==e0&&h[4*l+1]==e1&&h[4*l+2]==e2&&h[4*l+3]==e3) ? "ok" : "MISMATCH");
  }
}

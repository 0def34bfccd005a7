// Integer-pipe microbenchmark for the enumeration roofline (POPC / LOP3 / IMNMX
// rates per SM per clock on the box's B200, plus the candidate inner loop).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

// 8 independent POPC chains per thread.
__global__ void k_popc(const uint32_t* in, uint32_t* out, int iters, long long* cyc) {
  uint32_t v[8];
  for (int i = 0; i < 8; i++) v[i] = in[(threadIdx.x + i) & 255] + i;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) v[i] = __popc(v[i]) ^ v[(i + 1) & 7];
  }
  long long t1 = clock64();
  uint32_t s = 0;
  for (int i = 0; i < 8; i++) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// LOP3 only: 8 chains.
__global__ void k_lop3(const uint32_t* in, uint32_t* out, int iters, long long* cyc) {
  uint32_t v[8], a = in[threadIdx.x & 255], b = in[(threadIdx.x * 7) & 255];
  for (int i = 0; i < 8; i++) v[i] = in[(threadIdx.x + i) & 255] + i;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      uint32_t r;
      asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(r) : "r"(v[i]), "r"(a), "r"(b));
      v[i] = r;
    }
  }
  long long t1 = clock64();
  uint32_t s = 0;
  for (int i = 0; i < 8; i++) s += v[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// Candidate loop: H=8 heads in registers, tails broadcast from smem.
// per candidate: 2 LOP3 + POPC + 1/2 min3
__global__ void k_cand(const uint32_t* in, uint32_t* out, int iters, long long* cyc) {
  __shared__ uint2 tails[256];
  tails[threadIdx.x & 255] = make_uint2(in[threadIdx.x & 255], in[(threadIdx.x * 3) & 255]);
  __syncthreads();
  uint32_t hx[8], hz[8];
  for (int i = 0; i < 8; i++) { hx[i] = in[(threadIdx.x + i) & 255]; hz[i] = in[(threadIdx.x + 2 * i) & 255]; }
  int m = 1000, hits = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
    for (int t = 0; t < 256; t += 2) {
      uint4 tt = *reinterpret_cast<const uint4*>(&tails[t]);
#pragma unroll
      for (int i = 0; i < 8; i++) {
        int w0 = __popc((hx[i] ^ tt.x) | (hz[i] ^ tt.y));
        int w1 = __popc((hx[i] ^ tt.z) | (hz[i] ^ tt.w));
        m = min(m, min(w0, w1));
      }
      if (m < 2) { hits++; m = 1000; }
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = m + hits;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  int nsm = 0; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  uint32_t *in, *out; long long* cyc;
  CK(cudaMalloc(&in, 4096 * 4)); CK(cudaMalloc(&out, 1 << 24)); CK(cudaMalloc(&cyc, 1 << 16));
  uint32_t h[4096]; uint64_t s = 88172645463325252ull;
  for (int i = 0; i < 4096; i++) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = (uint32_t)s; }
  CK(cudaMemcpy(in, h, sizeof h, cudaMemcpyHostToDevice));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int threads = 256;
  for (int occ : {4, 8}) {
    int blocks = nsm * occ;
    struct { const char* name; void (*k)(const uint32_t*, uint32_t*, int, long long*); int iters; double ops_per_iter; } ks[] = {
      {"popc", k_popc, 20000, 8.0}, {"lop3", k_lop3, 20000, 8.0}, {"cand", k_cand, 200, 256.0 * 8}};
    for (auto& K : ks) {
      for (int rep = 0; rep < 3; rep++) {
        cudaEventRecord(e0);
        K.k<<<blocks, threads>>>(in, out, K.iters, cyc);
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        long long c[4096]; CK(cudaMemcpy(c, cyc, blocks * 8, cudaMemcpyDeviceToHost));
        double cmax = 0, csum = 0; for (int b = 0; b < blocks; b++) { cmax = c[b] > cmax ? c[b] : cmax; csum += c[b]; }
        double total_ops = (double)blocks * threads * K.iters * K.ops_per_iter;
        double per_s = total_ops / (ms * 1e-3);
        double clk_ghz = cmax / (ms * 1e6);
        printf("occ=%d %-5s %.3f ms  %.3e ops/s  %.2f ops/clk/SM (SM clk from clock64/event: %.3f GHz)\n",
               occ, K.name, ms, per_s, per_s / (nsm * clk_ghz * 1e9), clk_ghz);
      }
    }
  }
  return 0;
}

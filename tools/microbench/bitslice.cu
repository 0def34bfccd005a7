// Does a bit-sliced (LOP3 carry-save) candidate path add throughput next to the POPC path?
// The POPC path is XU-bound (1 POPC per candidate) and leaves the ALU pipe about a third idle.
// The bit-sliced path scores 32 candidates at once: lane-held tail planes (bit j of plane b =
// bit b of tail j), warp-uniform head masks, a carry-save count of the 32 fold planes and an
// add-constant carry test for count <= T. Each warp runs its role for a fixed clock budget and
// counts candidates, so the co-running rate of each role comes out directly.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ void csa(uint32_t& h, uint32_t& l, uint32_t a, uint32_t b, uint32_t c) {
  uint32_t u = a ^ b;
  h = (a & b) | (u & c);
  l = u ^ c;
}

// POPC role: 8 heads per lane, tails as warp-uniform LDS.128 broadcasts (two per load).
__device__ __forceinline__ long long role_popc(const uint2* tails, const uint32_t* in, long long budget, int& sink) {
  uint32_t hx[8], hz[8];
  for (int i = 0; i < 8; i++) { hx[i] = in[(threadIdx.x + i) & 255]; hz[i] = in[(threadIdx.x + 2 * i) & 255]; }
  int m = 1000, hits = 0;
  long long n = 0, t0 = clock64();
  while (clock64() - t0 < budget) {
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
    n += 256 * 8;
  }
  sink += m + hits;
  return n;
}

// Bit-sliced role: the lane holds 32 tails as 2 x 32 planes; per head, 16 broadcast LDS.128
// bring its 64 masks (0 or ~0 per bit position and component).
__device__ __forceinline__ long long role_bs(const uint4* masks, int nheads, const uint32_t* in, long long budget,
                                             uint32_t thr_k, int& sink) {
  uint32_t Tx[32], Tz[32];
#pragma unroll
  for (int b = 0; b < 32; b++) { Tx[b] = in[(threadIdx.x * 5 + b) & 4095]; Tz[b] = in[(threadIdx.x * 3 + 7 * b) & 4095]; }
  uint32_t kb[6];
#pragma unroll
  for (int k = 0; k < 6; k++) kb[k] = ((thr_k >> k) & 1) ? ~0u : 0u;
  uint32_t acc = 0; int hits = 0;
  long long n = 0, t0 = clock64();
  while (clock64() - t0 < budget) {
    for (int h = 0; h < nheads; h++) {
      const uint4* M = masks + h * 16;
      uint32_t ones = 0, twos = 0, fours = 0, eights = 0, s16a = 0, s16b = 0;
#pragma unroll
      for (int q = 0; q < 2; q++) {         // two halves of 16 planes
        uint32_t e8[2];
#pragma unroll
        for (int r = 0; r < 2; r++) {       // 8 planes each
          uint32_t f4[2];
#pragma unroll
          for (int s = 0; s < 2; s++) {     // 4 planes each
            int b0 = q * 16 + r * 8 + s * 4;
            uint4 mx = M[b0 / 4], mz = M[8 + b0 / 4];
            uint32_t u0 = (Tx[b0] ^ mx.x) | (Tz[b0] ^ mz.x);
            uint32_t u1 = (Tx[b0 + 1] ^ mx.y) | (Tz[b0 + 1] ^ mz.y);
            uint32_t u2 = (Tx[b0 + 2] ^ mx.z) | (Tz[b0 + 2] ^ mz.z);
            uint32_t u3 = (Tx[b0 + 3] ^ mx.w) | (Tz[b0 + 3] ^ mz.w);
            uint32_t ta, tb;
            csa(ta, ones, ones, u0, u1);
            csa(tb, ones, ones, u2, u3);
            csa(f4[s], twos, twos, ta, tb);
          }
          csa(e8[r], fours, fours, f4[0], f4[1]);
        }
        if (q == 0) csa(s16a, eights, eights, e8[0], e8[1]);
        else csa(s16b, eights, eights, e8[0], e8[1]);
      }
      uint32_t c16 = s16a ^ s16b, c32 = s16a & s16b;
      // count + K >= 64  <=>  count > T  (K = 63 - T): ripple the carry through the 6 bits
      uint32_t cy = ones & kb[0];
      cy = (twos & cy) | (kb[1] & (twos | cy));
      cy = (fours & cy) | (kb[2] & (fours | cy));
      cy = (eights & cy) | (kb[3] & (eights | cy));
      cy = (c16 & cy) | (kb[4] & (c16 | cy));
      cy = (c32 & cy) | (kb[5] & (c32 | cy));
      acc |= ~cy;
      if (acc) { hits++; acc = 0; }
    }
    n += (long long)nheads * 32;
  }
  sink += hits;
  return n;
}


// Packed bit-sliced role: 16 tails per lane, plane q holds symbol q (low half) and q + 16 (high
// half), so 2 x 16 plane registers; per head 8 broadcast LDS.128 bring 32 half-word masks.
__device__ __forceinline__ long long role_bs16(const uint4* masks, int nheads, const uint32_t* in, long long budget,
                                               uint32_t thr_k, int& sink) {
  uint32_t Px[16], Pz[16];
#pragma unroll
  for (int b = 0; b < 16; b++) { Px[b] = in[(threadIdx.x * 5 + b) & 4095]; Pz[b] = in[(threadIdx.x * 3 + 7 * b) & 4095]; }
  const uint32_t k0 = (thr_k & 1) ? 0xffffu : 0u, k1 = (thr_k & 2) ? 0xffffu : 0u, k2 = (thr_k & 4) ? 0xffffu : 0u,
                 k3 = (thr_k & 8) ? 0xffffu : 0u, k4 = (thr_k & 16) ? ~0u : 0u;
  uint32_t acc = 0; int hits = 0;
  long long n = 0, t0 = clock64();
  while (clock64() - t0 < budget) {
    for (int h = 0; h < nheads; h++) {
      const uint4* M = masks + h * 8;
      uint32_t ones = k0, twos = k1, fours = k2, eights = k3, s16 = 0;
      uint32_t e8[2];
#pragma unroll
      for (int r = 0; r < 2; r++) {
        uint32_t f4[2];
#pragma unroll
        for (int s = 0; s < 2; s++) {
          int b0 = r * 8 + s * 4;
          uint4 mx = M[b0 / 4], mz = M[4 + b0 / 4];
          uint32_t u0 = (Px[b0] ^ mx.x) | (Pz[b0] ^ mz.x);
          uint32_t u1 = (Px[b0 + 1] ^ mx.y) | (Pz[b0 + 1] ^ mz.y);
          uint32_t u2 = (Px[b0 + 2] ^ mx.z) | (Pz[b0 + 2] ^ mz.z);
          uint32_t u3 = (Px[b0 + 3] ^ mx.w) | (Pz[b0 + 3] ^ mz.w);
          uint32_t ta, tb;
          csa(ta, ones, ones, u0, u1);
          csa(tb, ones, ones, u2, u3);
          csa(f4[s], twos, twos, ta, tb);
        }
        csa(e8[r], fours, fours, f4[0], f4[1]);
      }
      csa(s16, eights, eights, e8[0], e8[1]);
      // fold the high half (symbols 16..31) into the low half: carry out of the 4-bit add
      uint32_t c = ones & (ones >> 16);
      c = (twos & c) | ((twos >> 16) & (twos | c));
      c = (fours & c) | ((fours >> 16) & (fours | c));
      c = (eights & c) | ((eights >> 16) & (eights | c));
      const uint32_t h16 = s16 >> 16;
      // pass iff at most one of {c, s16, h16, k4}
      const uint32_t two = (c & s16) | (h16 & (c | s16)) | (k4 & (c | s16 | h16));
      acc |= ~two & 0xffffu;
      if (acc) { hits++; acc = 0; }
    }
    n += (long long)nheads * 16;
  }
  sink += hits;
  return n;
}

template <int NB>
__global__ void __launch_bounds__(256, 3) k_mix(const uint32_t* in, const uint4* gmasks, uint32_t* out, long long budget,
                                                unsigned long long* cnt_p, unsigned long long* cnt_b) {
  __shared__ uint2 tails[256];
  __shared__ uint4 masks[64 * 16];
  tails[threadIdx.x & 255] = make_uint2(in[threadIdx.x & 255], in[(threadIdx.x * 3) & 255]);
  for (int i = threadIdx.x; i < 64 * 16; i += blockDim.x) masks[i] = gmasks[i];
  __syncthreads();
  int warp = threadIdx.x >> 5, sink = 0;
  if (warp < NB) {
    long long n = role_bs(masks, 64, in, budget, 63 - 9, sink);
    if ((threadIdx.x & 31) == 0) atomicAdd(cnt_b, (unsigned long long)n * 32);
  } else {
    long long n = role_popc(tails, in, budget, sink);
    if ((threadIdx.x & 31) == 0) atomicAdd(cnt_p, (unsigned long long)n * 32);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = sink;
}

template <int NB>
__global__ void __launch_bounds__(256, 4) k_mix4(const uint32_t* in, const uint4* gmasks, uint32_t* out, long long budget,
                                                 unsigned long long* cnt_p, unsigned long long* cnt_b) {
  __shared__ uint2 tails[256];
  __shared__ uint4 masks[64 * 16];
  tails[threadIdx.x & 255] = make_uint2(in[threadIdx.x & 255], in[(threadIdx.x * 3) & 255]);
  for (int i = threadIdx.x; i < 64 * 16; i += blockDim.x) masks[i] = gmasks[i];
  __syncthreads();
  int warp = threadIdx.x >> 5, sink = 0;
  if (warp < NB) {
    long long n = role_bs(masks, 64, in, budget, 63 - 9, sink);
    if ((threadIdx.x & 31) == 0) atomicAdd(cnt_b, (unsigned long long)n * 32);
  } else {
    long long n = role_popc(tails, in, budget, sink);
    if ((threadIdx.x & 31) == 0) atomicAdd(cnt_p, (unsigned long long)n * 32);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = sink;
}


template <int NB>
__global__ void __launch_bounds__(256, 4) k_mix16(const uint32_t* in, const uint4* gmasks, uint32_t* out, long long budget,
                                                  unsigned long long* cnt_p, unsigned long long* cnt_b) {
  __shared__ uint2 tails[256];
  __shared__ uint4 masks[64 * 16];
  tails[threadIdx.x & 255] = make_uint2(in[threadIdx.x & 255], in[(threadIdx.x * 3) & 255]);
  for (int i = threadIdx.x; i < 64 * 16; i += blockDim.x) masks[i] = gmasks[i];
  __syncthreads();
  int warp = threadIdx.x >> 5, sink = 0;
  if (warp < NB) {
    long long n = role_bs16(masks, 64, in, budget, 63 - 9, sink);
    if ((threadIdx.x & 31) == 0) atomicAdd(cnt_b, (unsigned long long)n * 32);
  } else {
    long long n = role_popc(tails, in, budget, sink);
    if ((threadIdx.x & 31) == 0) atomicAdd(cnt_p, (unsigned long long)n * 32);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = sink;
}

typedef void (*KFn)(const uint32_t*, const uint4*, uint32_t*, long long, unsigned long long*, unsigned long long*);

int main() {
  int nsm = 0; CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  uint32_t *in, *out; uint4* gm; unsigned long long* cnt;
  CK(cudaMalloc(&in, 4096 * 4)); CK(cudaMalloc(&out, 1 << 24)); CK(cudaMalloc(&gm, 64 * 16 * 16)); CK(cudaMalloc(&cnt, 16));
  static uint32_t h[4096]; uint64_t s = 88172645463325252ull;
  for (int i = 0; i < 4096; i++) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; h[i] = (uint32_t)s; }
  CK(cudaMemcpy(in, h, sizeof h, cudaMemcpyHostToDevice));
  static uint32_t mh[64 * 64];
  for (int i = 0; i < 64 * 64; i++) mh[i] = (h[(i * 11) & 4095] & 1) ? ~0u : 0u;
  CK(cudaMemcpy(gm, mh, sizeof mh, cudaMemcpyHostToDevice));
  const long long budget = 20000000;  // ~10 ms at 1.9 GHz
  struct { const char* name; KFn k; int occ; } ks[] = {
      {"popc-only occ4", k_mix4<0>, 4}, {"bs1/8 occ4", k_mix4<1>, 4}, {"bs2/8 occ4", k_mix4<2>, 4},
      {"popc-only occ3", k_mix<0>, 3}, {"bs1/8 occ3", k_mix<1>, 3}, {"bs2/8 occ3", k_mix<2>, 3},
      {"bs3/8 occ3", k_mix<3>, 3}, {"bs8/8 occ3", k_mix<8>, 3}, {"bs8/8 occ4", k_mix4<8>, 4},
      {"p16 1/8 occ4", k_mix16<1>, 4}, {"p16 2/8 occ4", k_mix16<2>, 4}, {"p16 3/8 occ4", k_mix16<3>, 4}, {"p16 8/8 occ4", k_mix16<8>, 4}};
  for (auto& K : ks) {
    cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, K.k);
    int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, K.k, 256, 0);
    for (int rep = 0; rep < 2; rep++) {
      CK(cudaMemset(cnt, 0, 16));
      K.k<<<nsm * occ, 256>>>(in, gm, out, budget, cnt, cnt + 1);
      CK(cudaDeviceSynchronize());
      unsigned long long c[2]; CK(cudaMemcpy(c, cnt, 16, cudaMemcpyDeviceToHost));
      double per_clk_p = (double)c[0] / nsm / budget, per_clk_b = (double)c[1] / nsm / budget;
      printf("%-16s regs=%d spill=%zu occ=%d  popc %.2f + bs %.2f = %.2f cand/clk/SM\n", K.name, fa.numRegs,
             (size_t)fa.localSizeBytes, occ, per_clk_p, per_clk_b, per_clk_p + per_clk_b);
    }
  }
  return 0;
}

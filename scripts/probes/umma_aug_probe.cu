// Micro-probe (sm_100a): a K=16 "augmentation" step of the attention S MMA that adds a per-key
// bias column to S = Q K^T: D[r][c] += sum_k Qa[r][k] Ka[c][k] with no-swizzle K-major operands,
// Qa broadcast to all 128 rows (SBO = 0) and Ka's second 8-column core matrix aliased onto the
// first (LBO = 0). Checks D[r][c] == Ka[c][0] + Ka[c][1] + Ka[c][2] for every row.
#include <cstdio>
#include <cstdlib>
#include <cmath>

#include "common.cuh"

using namespace psa;

PSA_DEV uint64_t desc_noswz(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  return d;  // layout type 0 = no swizzle
}

struct Sm {
  uint16_t qa[2][64];     // two 8x8 bf16 core matrices (128 B each)
  uint16_t ka[16][64];    // 16 groups of 8 keys x 8 bf16 (128 B each)
  uint64_t done;
  uint32_t tmem;
};

__global__ void aug_kernel(const uint16_t* ka_in, float* out, int variant) {
  __shared__ __align__(1024) Sm sm;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 128; i += blockDim.x) {
    const int cm = i / 64, e = i % 64, col = e % 8;
    // core matrix 0: rows identical, cols 0..2 = 1.0 ; core matrix 1 = 0
    sm.qa[cm][e] = (cm == 0 && col < 3) ? 0x3F80 : 0;
  }
  for (int i = threadIdx.x; i < 16 * 64; i += blockDim.x) sm.ka[i / 64][i % 64] = ka_in[i];
  if (threadIdx.x == 0) {
    mbar_init(&sm.done, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    tmem_alloc(&sm.tmem, 128);
    tmem_relinquish();
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = sm.tmem;
  if (warp == 0) {
    constexpr uint32_t idesc = umma_idesc_bf16(128, 128, false, false);
    // variant 0: LBO = K-direction stride, SBO = M/N-direction stride
    // variant 1: roles swapped
    const uint32_t qa_k = 128, qa_mn = 0, ka_k = 0, ka_mn = 128;
    uint64_t ad, bd;
    if (variant == 0) {
      ad = desc_noswz(smem_u32(sm.qa), qa_k, qa_mn);
      bd = desc_noswz(smem_u32(sm.ka), ka_k, ka_mn);
    } else {
      ad = desc_noswz(smem_u32(sm.qa), qa_mn, qa_k);
      bd = desc_noswz(smem_u32(sm.ka), ka_mn, ka_k);
    }
    if (elect_one()) {
      mma_bf16_ss(tmem, ad, bd, idesc, 0u);
      mma_commit(&sm.done);
    }
    __syncwarp();
  }
  mbar_wait(&sm.done, 0);
  tc_fence_after();
  // every warp of 4 reads its 32 lanes
  const int row = threadIdx.x;
  uint32_t v[32];
  for (int c = 0; c < 4; ++c) {
    tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c * 32, v);
    tmem_ld_wait(v);
    for (int e = 0; e < 32; ++e) out[row * 128 + c * 32 + e] = __uint_as_float(v[e]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 128);
  }
}

static uint16_t f2bf(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  return static_cast<uint16_t>((u + 0x7FFF + ((u >> 16) & 1)) >> 16);
}
static float bf2f(uint16_t b) {
  uint32_t u = static_cast<uint32_t>(b) << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

int main() {
  uint16_t ka[16 * 64];
  float expect[128];
  const double c = 1.4426950408889634 / sqrt(128.0);
  for (int key = 0; key < 128; ++key) {
    const int h = 1 + key % 4;
    const bool pad = key % 17 == 5;
    double b = -(h - 1) / c;
    uint16_t t[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (pad) {
      t[0] = f2bf(-1.2676506e30f);
    } else {
      t[0] = f2bf(static_cast<float>(b));
      double r = b - bf2f(t[0]);
      t[1] = f2bf(static_cast<float>(r));
      r -= bf2f(t[1]);
      t[2] = f2bf(static_cast<float>(r));
    }
    for (int k = 0; k < 8; ++k) ka[(key / 8) * 64 + (key % 8) * 8 + k] = t[k];
    expect[key] = static_cast<float>(double(bf2f(t[0])) + bf2f(t[1]) + bf2f(t[2]));
  }
  uint16_t* dka;
  float* dout;
  cudaMalloc(&dka, sizeof(ka));
  cudaMalloc(&dout, 128 * 128 * 4);
  cudaMemcpy(dka, ka, sizeof(ka), cudaMemcpyHostToDevice);
  static float h[128 * 128];
  for (int variant = 0; variant < 2; ++variant) {
    cudaMemset(dout, 0, 128 * 128 * 4);
    aug_kernel<<<1, 128>>>(dka, dout, variant);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("variant %d: CUDA error %s\n", variant, cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(h, dout, sizeof(h), cudaMemcpyDeviceToHost);
    int bad = 0;
    double worst = 0;
    for (int r = 0; r < 128; ++r)
      for (int k = 0; k < 128; ++k) {
        const double d = fabs(h[r * 128 + k] - expect[k]) / fmax(1.0, fabs(expect[k]));
        worst = fmax(worst, d);
        if (d > 1e-6) ++bad;
      }
    printf("variant %d: %d / 16384 mismatches, worst rel %.3g; D[0][0..3] = %g %g %g %g (exp %g %g %g %g)\n",
           variant, bad, worst, h[0], h[1], h[2], h[3], expect[0], expect[1], expect[2], expect[3]);
  }
  return 0;
}

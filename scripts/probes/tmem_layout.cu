// Probe: thread <-> (TMEM lane, column) mapping of tcgen05.ld shapes 16x256b / 16x128b / 16x64b.
#include <cstdio>
#include <cstdint>
__global__ void probe(int* out) {
  __shared__ uint32_t base;
  const int lane = threadIdx.x;
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"((uint32_t)__cvta_generic_to_shared(&base)));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncwarp();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t t = base;
  uint32_t v[8];
  for (int c = 0; c < 8; ++c) v[c] = lane * 100 + c;
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(t),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
  asm volatile("tcgen05.wait::st.sync.aligned;");
  uint32_t a[4], b[2], c1;
  asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];" : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]) : "r"(t));
  asm volatile("tcgen05.ld.sync.aligned.16x128b.x1.b32 {%0,%1}, [%2];" : "=r"(b[0]), "=r"(b[1]) : "r"(t));
  asm volatile("tcgen05.ld.sync.aligned.16x64b.x1.b32 {%0}, [%1];" : "=r"(c1) : "r"(t));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int r = 0; r < 4; ++r) out[lane * 8 + r] = a[r];
  out[lane * 8 + 4] = b[0]; out[lane * 8 + 5] = b[1]; out[lane * 8 + 6] = c1;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncwarp();
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(t));
}
int main() {
  int* d; cudaMalloc(&d, 32 * 8 * 4); cudaMemset(d, 0xff, 32 * 8 * 4);
  probe<<<1, 32>>>(d);
  int h[256]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  for (int l = 0; l < 32; ++l) {
    printf("t%2d 16x256b:", l);
    for (int r = 0; r < 4; ++r) printf(" (%d,%d)", h[l * 8 + r] / 100, h[l * 8 + r] % 100);
    printf("  16x128b: (%d,%d) (%d,%d)  16x64b: (%d,%d)\n", h[l*8+4]/100, h[l*8+4]%100, h[l*8+5]/100, h[l*8+5]%100, h[l*8+6]/100, h[l*8+6]%100);
  }
}

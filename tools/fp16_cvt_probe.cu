// Probe: how do the fp16 pack conversions treat values beyond +-65504 on sm_100a?
#include <cstdio>
#include <cstdint>
__global__ void k(float x, uint32_t *out) {
  uint32_t a, b, c, d;
  asm("cvt.rn.relu.f16x2.f32 %0, %1, %2;" : "=r"(a) : "f"(x), "f"(-x));
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(b) : "f"(x), "f"(-x));
  asm("cvt.rn.relu.satfinite.f16x2.f32 %0, %1, %2;" : "=r"(c) : "f"(x), "f"(-x));
  uint16_t h;
  asm("cvt.rn.f16.f32 %0, %1;" : "=h"(h) : "f"(x));
  d = h;
  out[0] = a; out[1] = b; out[2] = c; out[3] = d;
}
int main() {
  uint32_t *o; cudaMallocManaged(&o, 16);
  for (float x : {1000.0f, 70000.0f, 1e6f}) {
    k<<<1, 1>>>(x, o); cudaDeviceSynchronize();
    printf("x=%g relu=%08x plain=%08x relu_sat=%08x f16=%04x\n", x, o[0], o[1], o[2], o[3]);
  }
}

// Accuracy of tanh.approx.bf16x2 over every finite bf16 input vs RNE_bf16(tanh(x)) in fp64,
// and of the current path RNE_bf16(tanh.approx.f32(x)).
#include <cstdio>
#include <cmath>
#include <cstring>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void k(const uint16_t* in, uint16_t* o16, float* o32, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (2 * i + 1 >= n) return;
  uint32_t x = (uint32_t)in[2 * i] | ((uint32_t)in[2 * i + 1] << 16), y;
  asm("tanh.approx.bf16x2 %0, %1;" : "=r"(y) : "r"(x));
  o16[2 * i] = (uint16_t)(y & 0xFFFF);
  o16[2 * i + 1] = (uint16_t)(y >> 16);
  for (int j = 0; j < 2; ++j) {
    float f; uint32_t u = (uint32_t)in[2 * i + j] << 16; memcpy(&f, &u, 4);
    float t; asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(f));
    o32[2 * i + j] = t;
  }
}
static uint16_t rne(double v) { float f = (float)v; uint32_t u; memcpy(&u, &f, 4); u += 0x7FFF + ((u >> 16) & 1); return (uint16_t)(u >> 16); }
static double bf(uint16_t b) { uint32_t u = (uint32_t)b << 16; float f; memcpy(&f, &u, 4); return f; }
int main() {
  const int n = 65536;
  uint16_t* h = new uint16_t[n]; for (int i = 0; i < n; ++i) h[i] = (uint16_t)i;
  uint16_t *d, *o; float* o32;
  cudaMalloc(&d, 2 * n); cudaMalloc(&o, 2 * n); cudaMalloc(&o32, 4 * n);
  cudaMemcpy(d, h, 2 * n, cudaMemcpyHostToDevice);
  k<<<n / 256, 128>>>(d, o, o32, n);
  uint16_t* r = new uint16_t[n]; float* r32 = new float[n];
  cudaMemcpy(r, o, 2 * n, cudaMemcpyDeviceToHost); cudaMemcpy(r32, o32, 4 * n, cudaMemcpyDeviceToHost);
  int cnt = 0, neq16 = 0, neq32 = 0, maxulp16 = 0, maxulp32 = 0; double maxrel16 = 0, maxrel32 = 0;
  for (int i = 0; i < n; ++i) {
    double x = bf((uint16_t)i);
    if (!std::isfinite(x) || std::fabs(x) > 20) continue;
    ++cnt;
    double t = std::tanh(x);
    uint16_t want = rne(t);
    uint16_t g16 = r[i], g32 = rne(r32[i]);
    int u16 = std::abs((int)(int16_t)g16 - (int)(int16_t)want), u32 = std::abs((int)(int16_t)g32 - (int)(int16_t)want);
    if (g16 != want) { ++neq16; if (u16 > maxulp16) maxulp16 = u16; }
    if (g32 != want) { ++neq32; if (u32 > maxulp32) maxulp32 = u32; }
    if (t != 0) { maxrel16 = std::fmax(maxrel16, std::fabs(bf(g16) - t) / std::fabs(t)); maxrel32 = std::fmax(maxrel32, std::fabs(bf(g32) - t) / std::fabs(t)); }
  }
  printf("inputs %d | bf16x2: mismatches %d (max %d ulp) max rel err %.3e | f32->bf16: mismatches %d (max %d ulp) max rel err %.3e\n",
         cnt, neq16, maxulp16, maxrel16, neq32, maxulp32, maxrel32);
}

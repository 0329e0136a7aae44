// Per-SM throughput of the softmax's instruction classes on this GPU (one CTA per SM, W warps):
// MUFU.EX2, FFMA2, FADD2, F2FP (bf16x2 pack), FMNMX3 and the softmax pair mix
// (FFMA2 + 2 MUFU.EX2 + FADD2 + F2FP). Prints ops per clock per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/sfu_probe tools/sfu_probe.cu && /tmp/sfu_probe
#include <cstdio>
#include <cuda_bf16.h>

constexpr int ITERS = 4096, U = 16;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm volatile("{\n\t.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
               "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
               : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 d;
  asm volatile("{\n\t.reg .b64 ra, rb, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
               "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
               : "=f"(d.x), "=f"(d.y) : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float max3(float a, float b, float c) {
  float d;
  asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ unsigned pack(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<unsigned*>(&h);
}

template <int MODE>
__global__ void probe(float* out, long long* cyc, float seed) {
  float v[U];
  float2 w[U];
  unsigned p = 0;
  for (int i = 0; i < U; ++i) {
    v[i] = seed * (threadIdx.x + i);
    w[i] = make_float2(v[i], -v[i]);
  }
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < U; ++i) {
      if (MODE == 0) v[i] = ex2(v[i]);
      if (MODE == 1) w[i] = ffma2(w[i], w[(i + 1) % U], w[(i + 3) % U]);
      if (MODE == 2) w[i] = fadd2(w[i], w[(i + 5) % U]);
      if (MODE == 3) p ^= pack(v[i], v[(i + 1) % U]), v[i] += 1.f;
      if (MODE == 4) v[i] = max3(v[i], v[(i + 1) % U], v[(i + 2) % U]);
      if (MODE == 5) {  // softmax pair: x = s*sc - m (FFMA2), 2 ex2, sum (FADD2), pack (F2FP)
        const float2 x = ffma2(w[i], make_float2(seed, seed), make_float2(-seed, -seed));
        const float a = ex2(x.x), b = ex2(x.y);
        w[(i + 7) % U] = fadd2(w[(i + 7) % U], make_float2(a, b));
        p ^= pack(a, b);
      }
    }
  }
  const long long t1 = clock64();
  float acc = p;
  for (int i = 0; i < U; ++i) acc += v[i] + w[i].x + w[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, int warps, double ops_per_elem) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  probe<MODE><<<148, warps * 32>>>(out, cyc, 0.001f);
  probe<MODE><<<148, warps * 32>>>(out, cyc, 0.001f);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  const double ops = (double)warps * 32 * ITERS * U * ops_per_elem;
  printf("%-28s warps/SM %2d: %7.2f per clk per SM\n", name, warps, ops / (double)mx);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<0>("MUFU.EX2 (lanes)", w, 1);
    run<1>("FFMA2 (fp32 FMA lanes)", w, 2);
    run<2>("FADD2 (fp32 add lanes)", w, 2);
    run<3>("F2FP bf16x2 pack (instr lanes)", w, 1);
    run<4>("FMNMX3 (instr lanes)", w, 1);
    run<5>("softmax pair (P elements)", w, 2);
  }
  return 0;
}

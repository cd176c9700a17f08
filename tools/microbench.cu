// microbench.cu -- sm_100a issue-rate microbenchmarks for the roofline
// denominators of the walk kernel: INT32 IMAD / IADD3 /
// LOP3 / POPC / IDP4A, legacy tensor-core mma.sync (f16->f32 m16n8k16,
// s8->s32 m16n8k32), and shared-memory load bandwidth.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
//   tools/microbench > profiles/microbench_peaks.json
//
// Each kernel runs 8 independent dependency chains per thread over a full
// persistent grid (148 SMs x 32 warps), so the pipe, not latency, limits it.
// The SM clock is measured inside the run (clock64 vs globaltimer), so the
// per-SM-per-clock rates are clock-independent.
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                         \
  do {                                                                                \
    cudaError_t e = (x);                                                              \
    if (e != cudaSuccess) {                                                           \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      exit(1);                                                                        \
    }                                                                                 \
  } while (0)

constexpr int ITERS = 4096;
constexpr int CH = 8;

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// clock probe: spin for a fixed number of SM cycles; events give the time
__global__ void k_clock(unsigned long long cycles) {
  const long long c0 = clock64();
  while ((unsigned long long)(clock64() - c0) < cycles) {
  }
}

__global__ void k_imad(uint32_t* out, uint32_t a, uint32_t b) {
  uint32_t x[CH];
#pragma unroll
  for (int c = 0; c < CH; c++) x[c] = threadIdx.x + c;
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) x[c] = x[c] * a + b;
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s ^= x[c];
  if (s == 0x12345678u) out[0] = s;
}

__global__ void k_iadd3(uint32_t* out, uint32_t a, uint32_t b) {
  uint32_t x[CH];
#pragma unroll
  for (int c = 0; c < CH; c++) x[c] = threadIdx.x * (c + 1);
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(x[c]) : "r"(a), "r"(b));
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s ^= x[c];
  if (s == 0x12345678u) out[0] = s;
}

__global__ void k_lop3(uint32_t* out, uint32_t a, uint32_t b) {
  uint32_t x[CH];
#pragma unroll
  for (int c = 0; c < CH; c++) x[c] = threadIdx.x * (c + 3);
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[c]) : "r"(a), "r"(b));
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s ^= x[c];
  if (s == 0x12345678u) out[0] = s;
}

__global__ void k_popc(uint32_t* out, uint32_t a) {
  uint32_t x[CH];
#pragma unroll
  for (int c = 0; c < CH; c++) x[c] = threadIdx.x * 2654435761u + c;
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) asm volatile("popc.b32 %0, %0;" : "+r"(x[c]));
#pragma unroll
    for (int c = 0; c < CH; c++) x[c] += a;  // keep the value wide
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s ^= x[c];
  if (s == 0x12345678u) out[0] = s;
}

__global__ void k_dp4a(int* out, int a, int b) {
  int x[CH];
#pragma unroll
  for (int c = 0; c < CH; c++) x[c] = threadIdx.x + c;
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) x[c] = __dp4a(a, b ^ c, x[c]);
  }
  int s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s ^= x[c];
  if (s == 0x12345678) out[0] = s;
}

// mma.sync m16n8k16 f16 x f16 -> f32; CH independent accumulators
__global__ void k_hmma(float* out, uint32_t a0) {
  uint32_t A[4] = {a0, a0 ^ 1u, a0 ^ 2u, a0 ^ 3u};
  uint32_t B[2] = {a0 ^ 5u, a0 ^ 7u};
  float acc[CH][4];
#pragma unroll
  for (int c = 0; c < CH; c++)
#pragma unroll
    for (int r = 0; r < 4; r++) acc[c][r] = 0.f;
  for (int i = 0; i < ITERS / 4; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) {
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+f"(acc[c][0]), "+f"(acc[c][1]), "+f"(acc[c][2]), "+f"(acc[c][3])
          : "r"(A[0]), "r"(A[1]), "r"(A[2]), "r"(A[3]), "r"(B[0]), "r"(B[1]));
    }
  }
  float s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s += acc[c][0] + acc[c][3];
  if (s == 1234.5f) out[0] = s;
}

// mma.sync m16n8k32 s8 x s8 -> s32
__global__ void k_imma(int* out, uint32_t a0) {
  uint32_t A[4] = {a0, a0 ^ 1u, a0 ^ 2u, a0 ^ 3u};
  uint32_t B[2] = {a0 ^ 5u, a0 ^ 7u};
  int acc[CH][4];
#pragma unroll
  for (int c = 0; c < CH; c++)
#pragma unroll
    for (int r = 0; r < 4; r++) acc[c][r] = 0;
  for (int i = 0; i < ITERS / 4; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) {
      asm volatile(
          "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+r"(acc[c][0]), "+r"(acc[c][1]), "+r"(acc[c][2]), "+r"(acc[c][3])
          : "r"(A[0]), "r"(A[1]), "r"(A[2]), "r"(A[3]), "r"(B[0]), "r"(B[1]));
    }
  }
  int s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s += acc[c][0] + acc[c][3];
  if (s == 1234567) out[0] = s;
}

// shared-memory LDS.32 bandwidth, conflict-free (inline PTX: nothing to hoist)
__global__ void k_lds(uint32_t* out, int stride_mask) {
  __shared__ uint32_t buf[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) buf[i] = (i * 33u) & 4095u;
  __syncthreads();
  uint32_t x[CH];
#pragma unroll
  for (int c = 0; c < CH; c++) x[c] = (threadIdx.x + 32 * c) & 4095;
  const uint32_t base = (uint32_t)__cvta_generic_to_shared(buf);
  for (int i = 0; i < ITERS; i++) {
#pragma unroll
    for (int c = 0; c < CH; c++) {
      uint32_t v;
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(base + 4u * ((x[c] + threadIdx.x) & (uint32_t)stride_mask)));
      x[c] = v;
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH; c++) s ^= x[c];
  if (s == 0x12345678u) out[0] = s;
}

struct Res {
  double ms;
};

template <class F>
double timeit(F f) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  f();  // warm-up
  CK(cudaDeviceSynchronize());
  double best = 1e30;
  for (int r = 0; r < 5; r++) {
    CK(cudaEventRecord(a));
    f();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int dev = 0, sms = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  uint32_t* d_u;
  CK(cudaMalloc(&d_u, 64));

  const int threads = 256;
  const int blocks = sms * 8;  // 64 warps/SM
  const double lanes = double(blocks) * threads;

  // SM clock: a kernel spinning a known cycle count on every SM, timed by events
  const unsigned long long spin = 400000000ull;
  const double spin_ms = timeit([&] { k_clock<<<sms, 32>>>(spin); });
  const double mhz = double(spin) / (spin_ms * 1e-3) / 1e6;

  auto rate = [&](double ms, double ops_per_lane) { return lanes * ops_per_lane / (ms * 1e-3); };
  double t;
  t = timeit([&] { k_imad<<<blocks, threads>>>(d_u, 3u, 7u); });
  const double imad = rate(t, double(ITERS) * CH);
  t = timeit([&] { k_iadd3<<<blocks, threads>>>(d_u, 3u, 7u); });
  const double iadd = rate(t, double(ITERS) * CH * 2);  // 2 PTX adds (may fuse to 1 IADD3)
  t = timeit([&] { k_lop3<<<blocks, threads>>>(d_u, 3u, 7u); });
  const double lop3 = rate(t, double(ITERS) * CH);
  t = timeit([&] { k_popc<<<blocks, threads>>>(d_u, 3u); });
  const double popc = rate(t, double(ITERS) * CH);
  t = timeit([&] { k_dp4a<<<blocks, threads>>>((int*)d_u, 0x01020304, 0x05060708); });
  const double dp4a = rate(t, double(ITERS) * CH);
  t = timeit([&] { k_hmma<<<blocks, threads>>>((float*)d_u, 0x3c003c00u); });
  const double hmma_inst = double(blocks) * threads / 32 * (ITERS / 4) * CH / (t * 1e-3);  // warp-level mma/s
  t = timeit([&] { k_imma<<<blocks, threads>>>((int*)d_u, 0x01010101u); });
  const double imma_inst = double(blocks) * threads / 32 * (ITERS / 4) * CH / (t * 1e-3);
  t = timeit([&] { k_lds<<<blocks, threads>>>(d_u, 4095); });
  const double lds = rate(t, double(ITERS) * CH);  // 4-byte loads per second

  const double clk = mhz * 1e6;
  auto per_sm_clk = [&](double r) { return r / sms / clk; };
  printf("{\n");
  printf("  \"gpu\": \"%s\", \"sms\": %d, \"sm_mhz_measured\": %.1f,\n", prop.name, sms, mhz);
  printf("  \"imad_lanes_per_s\": %.4e, \"imad_lanes_per_clk_sm\": %.2f,\n", imad, per_sm_clk(imad));
  printf("  \"iadd_lanes_per_s\": %.4e, \"iadd_lanes_per_clk_sm\": %.2f,\n", iadd, per_sm_clk(iadd));
  printf("  \"lop3_lanes_per_s\": %.4e, \"lop3_lanes_per_clk_sm\": %.2f,\n", lop3, per_sm_clk(lop3));
  printf("  \"popc_lanes_per_s\": %.4e, \"popc_lanes_per_clk_sm\": %.2f,\n", popc, per_sm_clk(popc));
  printf("  \"dp4a_lanes_per_s\": %.4e, \"dp4a_lanes_per_clk_sm\": %.2f,\n", dp4a, per_sm_clk(dp4a));
  printf("  \"hmma_m16n8k16_f16f32_per_s\": %.4e, \"hmma_per_clk_sm\": %.3f, \"hmma_tflops\": %.1f,\n", hmma_inst,
         per_sm_clk(hmma_inst), hmma_inst * 2.0 * 16 * 8 * 16 / 1e12);
  printf("  \"imma_m16n8k32_s8s32_per_s\": %.4e, \"imma_per_clk_sm\": %.3f, \"imma_tops\": %.1f,\n", imma_inst,
         per_sm_clk(imma_inst), imma_inst * 2.0 * 16 * 8 * 32 / 1e12);
  printf("  \"lds32_per_s\": %.4e, \"lds32_lanes_per_clk_sm\": %.2f,\n", lds, per_sm_clk(lds));
  printf("  \"imad_tops\": %.3f,\n", imad * 2 / 1e12);
  printf("  \"note\": \"imad_tops = measured IMAD lanes/s x 2 ops (1 MAC = 2 INT32 ops); rates at the measured clock\"\n");
  printf("}\n");
  return 0;
}

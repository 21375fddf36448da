// Microbenchmark: TMEM as a lane-private operand store for the chemistry
// kernel (K1).  K1's lanes are cells and every mechanism index is
// warp-uniform, so an operand gather "row k of the 32 cells" is exactly a
// tcgen05.ld.32x32b (lane = cell, column = uniform).  Measures, with one
// 1024-thread CTA per SM on every SM:
//   * LDS row gathers (the current data path)           bytes/clk/SM
//   * tcgen05.ld 32x32b.x2 / .x4 / .x8                  bytes/clk/SM
//   * both at once (are the two data paths additive?)
//   * tcgen05.cp 32x128b.warpx4 (smem -> all four lane quarters)
// and checks the no-swizzle descriptor layout of the copy bit for bit.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_probe scripts/tmem_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x)                                                                    \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess) {                                                     \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      exit(1);                                                                   \
    }                                                                            \
  } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void tmem_alloc512(uint32_t* slot)
{
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(slot)));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_free512(uint32_t base)
{
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void ld2(uint32_t a, uint32_t& r0, uint32_t& r1)
{
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(a));
}
__device__ __forceinline__ void ld4(uint32_t a, uint32_t (&r)[4])
{
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
}
__device__ __forceinline__ void ld8(uint32_t a, uint32_t (&r)[8])
{
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                 "=r"(r[7])
               : "r"(a));
}
__device__ __forceinline__ void st2(uint32_t a, uint32_t r0, uint32_t r1)
{
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(a), "r"(r0), "r"(r1));
}
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// keep the compiler from reading the destination registers before the wait
#define PIN(x) asm volatile("" : "+r"(x))

__device__ __forceinline__ double d2(uint32_t lo, uint32_t hi) { return __hiloint2double((int)hi, (int)lo); }

// MODE 0: LDS rows; 1: LDTM x2; 2: LDTM x4; 3: LDTM x8; 4: half warps LDS, half LDTM x2;
// 5: every warp alternates LDS and LDTM x2 (same instruction stream)
template <int MODE, int B>
__global__ void __launch_bounds__(1024, 1) tp(double* out, long long* cyc, int iters)
{
  extern __shared__ __align__(16) double sm[];  // [256][32] rows
  __shared__ uint32_t tslot;
  const int w = threadIdx.x >> 5, c = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 256 * 32; i += 1024) sm[i] = 1.0 + i * 1e-9;
  if (w == 0) tmem_alloc512(&tslot);
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tb = tslot + ((uint32_t)((w & 3) * 32) << 16);
  // fill this warp's quarter (8 warps share a quarter: each writes 64 columns)
  for (int col = (w >> 2) * 64; col < (w >> 2) * 64 + 64; col += 2) {
    const double v = 1.0 + (col * 32 + c) * 1e-9;
    st2(tb + col, (uint32_t)__double2loint(v), (uint32_t)__double2hiint(v));
  }
  wait_st();
  fence_before();
  __syncthreads();
  fence_after();
  long long t0 = clock64();
  double acc = 0.0;
  uint32_t k = (uint32_t)(w * 5);
  const bool lds_warp = MODE == 0 || (MODE == 4 && (w & 4));
  for (int it = 0; it < iters; ++it) {
    if (lds_warp) {
#pragma unroll
      for (int b = 0; b < B; ++b) acc += sm[((k + 17 * b) & 255) * 32 + c];
    } else if (MODE == 1 || MODE == 4) {
      uint32_t r[B][2];
#pragma unroll
      for (int b = 0; b < B; ++b) ld2(tb + (((k + 17 * b) * 2) & 511), r[b][0], r[b][1]);
      wait_ld();
#pragma unroll
      for (int b = 0; b < B; ++b) {
        PIN(r[b][0]);
        PIN(r[b][1]);
        acc += d2(r[b][0], r[b][1]);
      }
    } else if (MODE == 2) {
      uint32_t r[B][4];
#pragma unroll
      for (int b = 0; b < B; ++b) ld4(tb + (((k + 17 * b) * 4) & 511), r[b]);
      wait_ld();
#pragma unroll
      for (int b = 0; b < B; ++b) {
#pragma unroll
        for (int q = 0; q < 4; ++q) PIN(r[b][q]);
        acc += d2(r[b][0], r[b][1]) + d2(r[b][2], r[b][3]);
      }
    } else if (MODE == 3) {
      uint32_t r[B][8];
#pragma unroll
      for (int b = 0; b < B; ++b) ld8(tb + (((k + 17 * b) * 8) & 511), r[b]);
      wait_ld();
#pragma unroll
      for (int b = 0; b < B; ++b) {
#pragma unroll
        for (int q = 0; q < 8; ++q) PIN(r[b][q]);
        acc += d2(r[b][0], r[b][1]) + d2(r[b][2], r[b][3]) + d2(r[b][4], r[b][5]) + d2(r[b][6], r[b][7]);
      }
    } else if (MODE == 5) {
      uint32_t r[B][2];
#pragma unroll
      for (int b = 0; b < B; ++b) ld2(tb + (((k + 17 * b) * 2) & 511), r[b][0], r[b][1]);
#pragma unroll
      for (int b = 0; b < B; ++b) acc += sm[((k + 13 * b) & 255) * 32 + c];
      wait_ld();
#pragma unroll
      for (int b = 0; b < B; ++b) {
        PIN(r[b][0]);
        PIN(r[b][1]);
        acc += d2(r[b][0], r[b][1]);
      }
    }
    k += 29;
  }
  fence_before();
  __syncthreads();
  long long t1 = clock64();
  fence_after();
  if (w == 0) tmem_free512(tslot);
  out[blockIdx.x * 1024 + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// UTCCP 32x128b.warpx4: NCP copies of 512 B (32 rows x 16 B) from shared
// memory, each replicated into the four lane quarters; then every warp
// checks its quarter against the source.
__global__ void __launch_bounds__(1024, 1) cp_probe(double* out, long long* cyc, int* bad, int ncp, int reps)
{
  extern __shared__ __align__(16) double sm[];  // ncp tiles x [32 rows][2 doubles]
  __shared__ uint32_t tslot;
  __shared__ __align__(8) unsigned long long mbar;
  const int w = threadIdx.x >> 5, c = threadIdx.x & 31;
  for (int i = threadIdx.x; i < ncp * 64; i += 1024) sm[i] = 1.0 + i + blockIdx.x * 1e-6;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (w == 0) tmem_alloc512(&tslot);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t base = tslot;
  long long t0 = clock64();
  uint32_t phase = 0;
  for (int r = 0; r < reps; ++r) {
    if (threadIdx.x == 0) {
      for (int i = 0; i < ncp; ++i) {
        const uint32_t sa = su32(sm + i * 64);
        // no-swizzle K-major: core matrices of 8 rows x 16 B; SBO (M stride
        // between core matrices) = 128 B, LBO unused (one 16-B column)
        uint64_t desc = (uint64_t)((sa >> 4) & 0x3FFF);
        desc |= (uint64_t)(128 >> 4) << 16;   // LBO
        desc |= (uint64_t)(128 >> 4) << 32;   // SBO
        desc |= (uint64_t)1 << 46;            // version (sm100)
        const uint32_t dst = base + (uint32_t)((i * 4) & 511);
        asm volatile("tcgen05.cp.cta_group::1.32x128b.warpx4 [%0], %1;" ::"r"(dst), "l"(desc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          su32(&mbar)));
    }
    // everyone waits for the copies
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
            su32(&mbar)),
        "r"(phase));
    phase ^= 1;
    fence_after();
  }
  long long t1 = clock64();
  // verify: quarter (w & 3) lane c column 4i.. = tile i row c
  const uint32_t tb = base + ((uint32_t)((w & 3) * 32) << 16);
  int nbad = 0;
  for (int i = (w >> 2); i < ncp && i < 128; i += 8) {
    uint32_t r[4];
    ld4(tb + (uint32_t)(i * 4), r);
    wait_ld();
#pragma unroll
    for (int q = 0; q < 4; ++q) PIN(r[q]);
    const double a = d2(r[0], r[1]), b = d2(r[2], r[3]);
    if (a != sm[i * 64 + c * 2] || b != sm[i * 64 + c * 2 + 1]) ++nbad;
  }
  if (nbad) atomicAdd(bad, nbad);
  fence_before();
  __syncthreads();
  fence_after();
  if (w == 0) tmem_free512(tslot);
  out[blockIdx.x] = (double)nbad;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE, int B>
void run_tp(const char* name, int nsm, double* dout, long long* dcyc, double bytes_per_warp_iter)
{
  const int iters = 4096;
  const size_t smem = 256 * 32 * 8 + 0;
  CK(cudaFuncSetAttribute(tp<MODE, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(120 << 10)));
  tp<MODE, B><<<nsm, 1024, 120 << 10>>>(dout, dcyc, 16);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  tp<MODE, B><<<nsm, 1024, 120 << 10>>>(dout, dcyc, iters);
  cudaEventRecord(e1);
  CK(cudaDeviceSynchronize());
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  long long h[1024];
  CK(cudaMemcpy(h, dcyc, nsm * sizeof(long long), cudaMemcpyDeviceToHost));
  double mx = 0, s = 0;
  for (int i = 0; i < nsm; ++i) {
    s += h[i];
    if (h[i] > mx) mx = h[i];
  }
  const double bytes_sm = bytes_per_warp_iter * 32.0 * iters;
  printf("%-34s B=%d  cyc(max) %9.0f  bytes/clk/SM %7.1f  (avg-cyc %7.1f)  %.3f ms  chip %.2f TB/s\n", name, B, mx,
         bytes_sm / mx, bytes_sm / (s / nsm), ms, bytes_sm * nsm / (ms * 1e-3) / 1e12);
  (void)smem;
}

int main()
{
  int dev = 0, nsm = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  double* dout;
  long long* dcyc;
  int* dbad;
  CK(cudaMalloc(&dout, (size_t)nsm * 1024 * sizeof(double)));
  CK(cudaMalloc(&dcyc, 1024 * sizeof(long long)));
  CK(cudaMalloc(&dbad, sizeof(int)));
  printf("SMs %d\n", nsm);
  // bytes moved per warp per iteration
  run_tp<0, 4>("LDS row (8 B/lane)", nsm, dout, dcyc, 4 * 256.0);
  run_tp<0, 8>("LDS row (8 B/lane)", nsm, dout, dcyc, 8 * 256.0);
  run_tp<1, 1>("LDTM 32x32b.x2 (8 B/lane)", nsm, dout, dcyc, 1 * 256.0);
  run_tp<1, 4>("LDTM 32x32b.x2 (8 B/lane)", nsm, dout, dcyc, 4 * 256.0);
  run_tp<1, 8>("LDTM 32x32b.x2 (8 B/lane)", nsm, dout, dcyc, 8 * 256.0);
  run_tp<2, 4>("LDTM 32x32b.x4 (16 B/lane)", nsm, dout, dcyc, 4 * 512.0);
  run_tp<3, 2>("LDTM 32x32b.x8 (32 B/lane)", nsm, dout, dcyc, 2 * 1024.0);
  run_tp<3, 4>("LDTM 32x32b.x8 (32 B/lane)", nsm, dout, dcyc, 4 * 1024.0);
  run_tp<4, 4>("half LDS / half LDTM.x2", nsm, dout, dcyc, 4 * 256.0);
  run_tp<5, 4>("each warp LDS + LDTM.x2", nsm, dout, dcyc, 8 * 256.0);

  for (int ncp : {64, 128}) {
    const int reps = 64;
    CK(cudaFuncSetAttribute(cp_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(ncp * 512)));
    CK(cudaMemset(dbad, 0, sizeof(int)));
    cp_probe<<<nsm, 1024, ncp * 512>>>(dout, dcyc, dbad, ncp, reps);
    CK(cudaDeviceSynchronize());
    long long h[1024];
    int bad;
    CK(cudaMemcpy(h, dcyc, nsm * sizeof(long long), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&bad, dbad, sizeof(int), cudaMemcpyDeviceToHost));
    double mx = 0;
    for (int i = 0; i < nsm; ++i)
      if (h[i] > mx) mx = h[i];
    printf("UTCCP 32x128b.warpx4 x%3d: %8.1f clk per batch, %6.1f clk/copy, smem-read %6.1f B/clk, layout mismatches %d\n",
           ncp, mx / reps, mx / reps / ncp, 512.0 * ncp * reps / mx, bad);
  }
  printf("done\n");
  return 0;
}

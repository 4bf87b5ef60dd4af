// gather_probe.cu — microbenchmark for the next mstream_kernel candidate:
// gathering 64-byte factor rows (rank 16, float32) with per-lane LDG.128
// (what mstream_kernel does today: one L1 data-pipe wavefront per distinct
// 128-byte line, the pipe the kernel is bound by) versus TMA
// `tile::gather4` (4 rows per instruction into shared memory, bypassing the
// LSU pipe; rows then read back with LDS.128 at 0.5 wavefront per row).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_probe \
//        tools/gather_probe.cu -L/usr/local/cuda/lib64/stubs -lcuda
//   ./gather_probe <variant: ldg|tex4|tex2|tex1|tma> <skew: 0 uniform, 1 skewed> [box_rows] [table rows]
//
// Not part of the product: a measurement tool for DESIGN.md §4.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <vector>
#include <random>
#include <cmath>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

constexpr int R = 16;            // floats per row (64 bytes)
constexpr int THREADS = 256;

// (A) LDG: 4 lanes per row, float4 each; a warp instruction gathers 8 rows.
__global__ void __launch_bounds__(THREADS, 3) ldg_kernel(const float* __restrict__ F, const unsigned* __restrict__ idx,
                                                         long long n, float* out) {
  const int lane = threadIdx.x & 31, g = lane >> 2, gl = lane & 3;
  const long long w0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = (gridDim.x * (long long)blockDim.x) >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  // each warp owns chunks of 256 rows: per step 8 rows x U=4 in flight
  for (long long c = w0 * 256; c < n; c += nw * 256) {
#pragma unroll 1
    for (int j = 0; j < 256; j += 32) {
      unsigned r[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) r[u] = __ldg(idx + c + j + u * 8 + g);
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldg(reinterpret_cast<const float4*>(F + (size_t)r[u] * R) + gl);
#pragma unroll
      for (int u = 0; u < 4; ++u) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

// (C) texture path: the same rows fetched with tex1Dfetch<float4> from a linear
// texture object (the TEX data pipe of the L1), all of them (TEXF = 4) or
// TEXF of every 4 row gathers with the others on LDG (do the two pipes add up?).
template <int TEXF>
__global__ void __launch_bounds__(THREADS, 3) tex_kernel(cudaTextureObject_t tex, const float* __restrict__ F,
                                                         const unsigned* __restrict__ idx, long long n, float* out) {
  const int lane = threadIdx.x & 31, g = lane >> 2, gl = lane & 3;
  const long long w0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = (gridDim.x * (long long)blockDim.x) >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  for (long long c = w0 * 256; c < n; c += nw * 256) {
#pragma unroll 1
    for (int j = 0; j < 256; j += 32) {
      unsigned r[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) r[u] = __ldg(idx + c + j + u * 8 + g);
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (u < TEXF)
          v[u] = tex1Dfetch<float4>(tex, static_cast<int>(r[u] * 4 + gl));
        else
          v[u] = __ldg(reinterpret_cast<const float4*>(F + (size_t)r[u] * R) + gl);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

// (B) TMA gather4: per warp a ring of S stages of 32 rows (2 KB); lanes 0..7
// each issue one gather4 (4 rows) per stage; the warp waits on the stage's
// mbarrier and reads the 32 rows with LDS.128 (lane: row lane/4 + 8k, quarter lane%4).
constexpr int STAGES = 6;
constexpr int STAGE_ROWS = 32;
constexpr int STAGE_BYTES = STAGE_ROWS * R * 4;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

__global__ void __launch_bounds__(THREADS, 1) tma_kernel(const __grid_constant__ CUtensorMap tm, const unsigned* __restrict__ idx,
                                                         long long n, float* out, int box_rows) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ __align__(8) unsigned long long bar[THREADS / 32][STAGES];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* ring = smem + warp * STAGES * STAGE_BYTES;
  if (lane < STAGES) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(smem_u32(&bar[warp][lane])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const long long w0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nw = (gridDim.x * (long long)blockDim.x) >> 5;
  // stage sequence of this warp: chunk w0, w0+nw, ... (32 rows each)
  const long long nchunks = n / STAGE_ROWS;
  auto issue = [&](long long ch, int st) {
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(smem_u32(&bar[warp][st])), "r"(STAGE_BYTES) : "memory");
    __syncwarp();
    if (lane < 8) {
      const uint4 r4 = __ldg(reinterpret_cast<const uint4*>(idx + ch * STAGE_ROWS) + lane);
      const unsigned dst = smem_u32(ring + st * STAGE_BYTES + lane * 4 * R * 4);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
          :: "r"(dst), "l"(reinterpret_cast<uint64_t>(&tm)), "r"(smem_u32(&bar[warp][st])),
             "r"(0), "r"(r4.x), "r"(r4.y), "r"(r4.z), "r"(r4.w) : "memory");
    }
  };
  float4 acc = make_float4(0, 0, 0, 0);
  long long ch = w0;
  for (int s = 0; s < STAGES; ++s) if (ch + (long long)s * nw < nchunks) issue(ch + (long long)s * nw, s);
  unsigned phase = 0;
  int st = 0;
  for (; ch < nchunks; ch += nw) {
    // wait for stage st
    const unsigned b = smem_u32(&bar[warp][st]);
    unsigned done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done) : "r"(b), "r"(phase) : "memory");
    const float4* rows = reinterpret_cast<const float4*>(ring + st * STAGE_BYTES);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float4 v = rows[(lane >> 2) * 4 + k * 32 + (lane & 3)];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    __syncwarp();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const long long nx = ch + (long long)STAGES * nw;
    if (nx < nchunks) issue(nx, st);
    if (++st == STAGES) { st = 0; phase ^= 1; }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  const char* variant = argc > 1 ? argv[1] : "ldg";
  const int skew = argc > 2 ? atoi(argv[2]) : 0;
  const int box_rows = argc > 3 ? atoi(argv[3]) : 1;
  // table rows: default = cfg2 mode-0 factor, 12.8 MB (L2 resident); 20000000 = cfg5 mode-1 factor,
  // 1.28 GB (random 64-byte rows from DRAM)
  const long long rows_tab = argc > 4 ? atoll(argv[4]) : 200000;
  const long long n = 100000000;           // 2 gathered rows x 50M elements (cfg2, one mode)
  std::vector<float> hF(rows_tab * R);
  for (size_t i = 0; i < hF.size(); ++i) hF[i] = (float)((i * 2654435761u) % 1000) * 1e-3f;
  std::vector<unsigned> hI(n);
  std::mt19937_64 rng(7);
  std::uniform_real_distribution<double> U01(0.0, 1.0);
  for (long long i = 0; i < n; ++i) {
    double u = U01(rng);
    hI[i] = skew ? (unsigned)std::min<double>(rows_tab - 1, std::floor(rows_tab * u * u * u)) : (unsigned)(u * rows_tab);
  }
  double ref = 0;
  for (long long i = 0; i < n; ++i) { const float* r = &hF[(size_t)hI[i] * R]; for (int q = 0; q < R; ++q) ref += r[q]; }
  float *F, *out; unsigned* I;
  CK(cudaMalloc(&F, hF.size() * 4)); CK(cudaMalloc(&I, n * 4));
  CK(cudaMemcpy(F, hF.data(), hF.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(I, hI.data(), n * 4, cudaMemcpyHostToDevice));
  int sms = 0; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int blocks = strcmp(variant, "tma") == 0 ? sms : sms * 3;
  CK(cudaMalloc(&out, (size_t)blocks * THREADS * 4));
  CUtensorMap tm;
  if (strcmp(variant, "tma") == 0) {
    void* fn = nullptr; cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    cuuint64_t gdim[2] = {(cuuint64_t)R, (cuuint64_t)rows_tab};
    cuuint64_t gstr[1] = {(cuuint64_t)R * 4};
    cuuint32_t box[2] = {(cuuint32_t)R, (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = ((EncodeFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, F, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode rc=%d\n", (int)r);
    if (r) return 1;
    CK(cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * STAGES * STAGE_BYTES));
  }
  cudaTextureObject_t tex = 0;
  if (strncmp(variant, "tex", 3) == 0) {
    cudaResourceDesc rd{};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = F;
    rd.res.linear.desc = cudaCreateChannelDesc<float4>();
    rd.res.linear.sizeInBytes = hF.size() * 4;
    cudaTextureDesc td{};
    td.readMode = cudaReadModeElementType;
    CK(cudaCreateTextureObject(&tex, &rd, &td, nullptr));
  }
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  auto launch = [&]() {
    if (strcmp(variant, "tex4") == 0)
      tex_kernel<4><<<blocks, THREADS>>>(tex, F, I, n, out);
    else if (strcmp(variant, "tex2") == 0)
      tex_kernel<2><<<blocks, THREADS>>>(tex, F, I, n, out);
    else if (strcmp(variant, "tex1") == 0)
      tex_kernel<1><<<blocks, THREADS>>>(tex, F, I, n, out);
    else if (strcmp(variant, "tma") == 0)
      tma_kernel<<<blocks, THREADS, 8 * STAGES * STAGE_BYTES>>>(tm, I, n, out, box_rows);
    else
      ldg_kernel<<<blocks, THREADS>>>(F, I, n, out);
  };
  float best = 1e30f;
  for (int it = 0; it < 8; ++it) {
    CK(cudaEventRecord(a)); launch(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    CK(cudaGetLastError());
    float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (it >= 2) best = std::min(best, ms);
  }
  std::vector<float> ho((size_t)blocks * THREADS);
  CK(cudaMemcpy(ho.data(), out, ho.size() * 4, cudaMemcpyDeviceToHost));
  double s = 0; for (float v : ho) s += v;
  printf("variant=%s skew=%d box_rows=%d table_rows=%lld rows=%lld best_ms=%.4f Grows/s=%.1f sum_rel_err=%.2e\n", variant, skew, box_rows, rows_tab, n, best,
         n / (best * 1e-3) / 1e9, std::fabs(s - ref) / ref);
  return 0;
}

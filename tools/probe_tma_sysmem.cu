// Probe: can sm_100a bulk-async copies (cp.async.bulk, the TMA engine) move
// data between mapped pinned host memory and shared memory at host-link
// speed, with few CTAs?  If so, the zero-copy transport's fetch / gather /
// stage could run on TMA instead of thread loads and stores (which need many
// warps in flight) or copy engines.  Prints JSON lines:
//   tma_load   host -> smem (bulk loads, mbarrier complete_tx, a ring of stages)
//   tma_store  smem -> host (bulk stores, bulk_group)
//   tma_both   half the CTAs load, half store (both link directions)
//   ldg_load   host -> registers with ld.global.cv.v4 (the current ZC gather)
//   stg_store  registers -> host with st.global.v4 (the current ZC stage)
//   ce_h2d / ce_d2h  cudaMemcpyAsync, for reference
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/probe_tma_sysmem tools/probe_tma_sysmem.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      fprintf(stderr, "%s failed: %s (line %d)\n", #x, cudaGetErrorString(e_), __LINE__); \
      exit(1);                                                                         \
    }                                                                                  \
  } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void bulk_load(void* smem, const void* gmem, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(smem)),
      "l"(gmem), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void bulk_store(void* gmem, const void* smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gmem),
               "r"(smem_u32(smem)), "r"(bytes)
               : "memory");
}

// Each CTA streams its share of [0, total) in chunks of `chunk` bytes through
// `stages` shared-memory buffers.  One thread drives the engine.
template <int kStages>
__global__ void tma_load_kernel(const char* __restrict__ src, size_t total, uint32_t chunk,
                                unsigned long long* sink) {
  extern __shared__ __align__(128) char smem[];
  __shared__ uint64_t bars[kStages];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const size_t nchunks = total / chunk;
  uint32_t phase[kStages] = {};
  size_t issued = 0, done = 0;
  unsigned long long acc = 0;
  // chunks blockIdx.x, blockIdx.x + gridDim.x, ...
  size_t next = blockIdx.x;
  for (int s = 0; s < kStages && next < nchunks; ++s, next += gridDim.x, ++issued) {
    mbar_expect_tx(&bars[s], chunk);
    bulk_load(smem + (size_t)s * chunk, src + next * chunk, chunk, &bars[s]);
  }
  int s = 0;
  while (done < issued) {
    mbar_wait(&bars[s], phase[s]);
    phase[s] ^= 1;
    acc += *(volatile unsigned long long*)(smem + (size_t)s * chunk);  // touch it
    ++done;
    if (next < nchunks) {
      mbar_expect_tx(&bars[s], chunk);
      bulk_load(smem + (size_t)s * chunk, src + next * chunk, chunk, &bars[s]);
      next += gridDim.x;
      ++issued;
    }
    s = (s + 1) % kStages;
  }
  if (acc == 0x12345) *sink = acc;
}

template <int kStages>
__global__ void tma_store_kernel(char* __restrict__ dst, size_t total, uint32_t chunk) {
  extern __shared__ __align__(128) char smem[];
  if (threadIdx.x != 0) return;
  for (uint32_t i = 0; i < chunk * kStages; i += 16) *(uint4*)(smem + i) = make_uint4(i, 1, 2, 3);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const size_t nchunks = total / chunk;
  int inflight = 0, s = 0;
  for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    if (inflight == kStages) {  // keep at most kStages bulk groups reading smem
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kStages - 1) : "memory");
      --inflight;
    }
    bulk_store(dst + c * chunk, smem + (size_t)s * chunk, chunk);
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    ++inflight;
    s = (s + 1) % kStages;
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void ldg_kernel(const uint4* __restrict__ src, size_t n16, unsigned long long* sink) {
  unsigned long long acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16;
       i += (size_t)gridDim.x * blockDim.x) {
    uint4 v;
    asm volatile("ld.global.cv.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(src + i));
    acc += v.x;
  }
  if (acc == 0x12345) *sink = acc;
}

// 256-bit stores / loads (sm_100: STG.E.ENL2.256 / LDG.E.ENL2.256), 32 B per thread
__global__ void stg256_kernel(float* __restrict__ dst, size_t n32) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n32;
       i += (size_t)gridDim.x * blockDim.x) {
    const float v = (float)i;
    asm volatile("st.global.v8.f32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(dst + i * 8), "f"(v)
                 : "memory");
  }
}

__global__ void ldg256_kernel(const float* __restrict__ src, size_t n32, unsigned long long* sink) {
  float acc = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n32;
       i += (size_t)gridDim.x * blockDim.x) {
    float a0, a1, a2, a3, a4, a5, a6, a7;
    asm volatile("ld.global.volatile.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(a0), "=f"(a1), "=f"(a2), "=f"(a3), "=f"(a4), "=f"(a5), "=f"(a6), "=f"(a7)
                 : "l"(src + i * 8));
    acc += a0 + a7;
  }
  if (acc == 12345.f) *sink = 1;
}

__global__ void stg_kernel(uint4* __restrict__ dst, size_t n16) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16;
       i += (size_t)gridDim.x * blockDim.x)
    dst[i] = make_uint4((uint32_t)i, 1, 2, 3);
}

template <int kStages>
__global__ void tma_both_kernel(const char* src, char* dst, size_t total, uint32_t chunk,
                                unsigned long long* sink) {
  // even CTAs load, odd CTAs store (grid is even)
  extern __shared__ __align__(128) char smem[];
  if (blockIdx.x % 2 == 0) {
    __shared__ uint64_t bars[kStages];
    if (threadIdx.x != 0) return;
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const size_t nchunks = total / chunk;
    const int me = blockIdx.x / 2, nb = gridDim.x / 2;
    uint32_t phase[kStages] = {};
    size_t issued = 0, done = 0, next = me;
    unsigned long long acc = 0;
    for (int s = 0; s < kStages && next < nchunks; ++s, next += nb, ++issued) {
      mbar_expect_tx(&bars[s], chunk);
      bulk_load(smem + (size_t)s * chunk, src + next * chunk, chunk, &bars[s]);
    }
    int s = 0;
    while (done < issued) {
      mbar_wait(&bars[s], phase[s]);
      phase[s] ^= 1;
      acc += *(volatile unsigned long long*)(smem + (size_t)s * chunk);
      ++done;
      if (next < nchunks) {
        mbar_expect_tx(&bars[s], chunk);
        bulk_load(smem + (size_t)s * chunk, src + next * chunk, chunk, &bars[s]);
        next += nb;
        ++issued;
      }
      s = (s + 1) % kStages;
    }
    if (acc == 0x12345) *sink = acc;
  } else {
    if (threadIdx.x != 0) return;
    for (uint32_t i = 0; i < chunk * kStages; i += 16) *(uint4*)(smem + i) = make_uint4(i, 1, 2, 3);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    const size_t nchunks = total / chunk;
    const int me = blockIdx.x / 2, nb = gridDim.x / 2;
    int inflight = 0, s = 0;
    for (size_t c = me; c < nchunks; c += nb) {
      if (inflight == kStages) {
        asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(kStages - 1) : "memory");
        --inflight;
      }
      bulk_store(dst + c * chunk, smem + (size_t)s * chunk, chunk);
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      ++inflight;
      s = (s + 1) % kStages;
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

template <typename F>
float time_ms(F&& launch, int iters) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  launch();
  CK(cudaDeviceSynchronize());
  CK(cudaEventRecord(a));
  for (int i = 0; i < iters; ++i) launch();
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  CK(cudaGetLastError());
  return ms / iters;
}

int main(int argc, char** argv) {
  const size_t total = argc > 1 ? strtoull(argv[1], nullptr, 10) : (512ull << 20);
  char *h_src, *h_dst, *d_buf;
  CK(cudaHostAlloc(&h_src, total, cudaHostAllocMapped | cudaHostAllocPortable));
  CK(cudaHostAlloc(&h_dst, total, cudaHostAllocMapped | cudaHostAllocPortable));
  CK(cudaMalloc(&d_buf, total));
  for (size_t i = 0; i < total; i += 4096) h_src[i] = (char)i;
  char *dv_src, *dv_dst;
  CK(cudaHostGetDevicePointer((void**)&dv_src, h_src, 0));
  CK(cudaHostGetDevicePointer((void**)&dv_dst, h_dst, 0));
  unsigned long long* sink;
  CK(cudaMalloc(&sink, 8));
  const int iters = 3;
  constexpr int kStages = 4;
  const int grids[] = {1, 2, 4, 8, 16, 32, 64, 148};
  const uint32_t chunks[] = {16384, 32768, 49152};
  const bool load_only = getenv("PROBE_LOAD_ONLY") != nullptr;
  for (uint32_t chunk : chunks) {
    if (load_only) break;
    const size_t smem = (size_t)chunk * kStages;
    CK(cudaFuncSetAttribute(tma_load_kernel<kStages>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaFuncSetAttribute(tma_store_kernel<kStages>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaFuncSetAttribute(tma_both_kernel<kStages>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    for (int g : grids) {
      float ms = time_ms([&] { tma_load_kernel<kStages><<<g, 32, smem>>>(dv_src, total, chunk, sink); }, iters);
      printf("{\"probe\": \"tma_load\", \"ctas\": %d, \"chunk\": %u, \"stages\": %d, \"gbs\": %.2f}\n", g, chunk,
             kStages, total / ms / 1e6);
      ms = time_ms([&] { tma_store_kernel<kStages><<<g, 32, smem>>>(dv_dst, total, chunk); }, iters);
      printf("{\"probe\": \"tma_store\", \"ctas\": %d, \"chunk\": %u, \"stages\": %d, \"gbs\": %.2f}\n", g, chunk,
             kStages, total / ms / 1e6);
      if (g >= 2) {
        ms = time_ms([&] { tma_both_kernel<kStages><<<g, 32, smem>>>(dv_src, dv_dst, total, chunk, sink); }, iters);
        printf("{\"probe\": \"tma_both\", \"ctas\": %d, \"chunk\": %u, \"stages\": %d, \"gbs_total\": %.2f}\n", g,
               chunk, kStages, 2 * total / ms / 1e6);
      }
      fflush(stdout);
    }
  }
  for (int g : grids) {
    if (load_only) break;
    float ms = time_ms([&] { ldg_kernel<<<g * 4, 512>>>((const uint4*)dv_src, total / 16, sink); }, iters);
    printf("{\"probe\": \"ldg_load\", \"ctas\": %d, \"threads\": 512, \"gbs\": %.2f}\n", g * 4, total / ms / 1e6);
    ms = time_ms([&] { stg_kernel<<<g * 4, 512>>>((uint4*)dv_dst, total / 16); }, iters);
    printf("{\"probe\": \"stg_store\", \"ctas\": %d, \"threads\": 512, \"gbs\": %.2f}\n", g * 4, total / ms / 1e6);
    fflush(stdout);
  }
  // under load: copy engines stream H2D and D2H on two other streams while
  // the SM / TMA store (or load) runs - the pipeline's live condition
  {
    const size_t big = 256ull << 20;
    char *h_a, *h_b, *d_a, *d_b;
    CK(cudaHostAlloc(&h_a, big, cudaHostAllocDefault));
    CK(cudaHostAlloc(&h_b, big, cudaHostAllocDefault));
    CK(cudaMalloc(&d_a, big));
    CK(cudaMalloc(&d_b, big));
    cudaStream_t sh, sd, sk;
    CK(cudaStreamCreateWithFlags(&sh, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&sd, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&sk, cudaStreamNonBlocking));
    const size_t part = 64ull << 20;  // kernel-side bytes per measurement
    auto under = [&](const char* name, int ctas, auto&& launch) {
      for (const char* load : {"none", "both"}) {
        CK(cudaDeviceSynchronize());
        if (load[0] == 'b')
          for (int i = 0; i < 12; ++i) {
            CK(cudaMemcpyAsync(d_a, h_a, big, cudaMemcpyHostToDevice, sh));
            CK(cudaMemcpyAsync(h_b, d_b, big, cudaMemcpyDeviceToHost, sd));
          }
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        launch(sk);
        CK(cudaGetLastError());
        CK(cudaEventRecord(a, sk));
        for (int i = 0; i < 5; ++i) launch(sk);
        CK(cudaEventRecord(b, sk));
        CK(cudaEventSynchronize(b));
        float ms = 0;
        CK(cudaEventElapsedTime(&ms, a, b));
        printf("{\"probe\": \"%s_under_load\", \"ctas\": %d, \"load\": \"%s\", \"gbs\": %.2f}\n", name,
               ctas, load, 5 * part / ms / 1e6);
        fflush(stdout);
        CK(cudaDeviceSynchronize());
      }
    };
    for (int g : {16, 64, 256}) under("stg_store", g, [&](cudaStream_t st) { stg_kernel<<<g, 512, 0, st>>>((uint4*)dv_dst, part / 16); });
    for (int g : {16, 64, 256}) under("ldg_load", g, [&](cudaStream_t st) { ldg_kernel<<<g, 512, 0, st>>>((const uint4*)dv_src, part / 16, sink); });
    for (int g : {16, 64, 256}) under("stg256_store", g, [&](cudaStream_t st) { stg256_kernel<<<g, 512, 0, st>>>((float*)dv_dst, part / 32); });
    for (int g : {16, 64, 256}) under("ldg256_load", g, [&](cudaStream_t st) { ldg256_kernel<<<g, 512, 0, st>>>((const float*)dv_src, part / 32, sink); });
    const uint32_t chunk = 32768;
    const size_t smem = (size_t)chunk * kStages;
    CK(cudaFuncSetAttribute(tma_load_kernel<kStages>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    CK(cudaFuncSetAttribute(tma_store_kernel<kStages>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    for (int g : {1, 4, 16}) under("tma_store", g, [&](cudaStream_t st) { tma_store_kernel<kStages><<<g, 32, smem, st>>>(dv_dst, part, chunk); });
    for (int g : {1, 4, 16}) under("tma_load", g, [&](cudaStream_t st) { tma_load_kernel<kStages><<<g, 32, smem, st>>>(dv_src, part, chunk, sink); });
  }
  float ms = time_ms([&] { CK(cudaMemcpyAsync(d_buf, h_src, total, cudaMemcpyHostToDevice)); }, iters);
  printf("{\"probe\": \"ce_h2d\", \"gbs\": %.2f}\n", total / ms / 1e6);
  ms = time_ms([&] { CK(cudaMemcpyAsync(h_dst, d_buf, total, cudaMemcpyDeviceToHost)); }, iters);
  printf("{\"probe\": \"ce_d2h\", \"gbs\": %.2f}\n", total / ms / 1e6);
  return 0;
}

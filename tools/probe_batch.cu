// Probe: does one stream overlap the two PCIe directions when the H2D and D2H
// copies are issued as ONE cudaMemcpyBatchAsync?  (If so, a single in-order
// stream per rank can software-pipeline bucket k's gather (H2D) with bucket
// k+1's stage (D2H) - the DDP join-stream mode runs on one stream.)
// Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o tools/probe_batch tools/probe_batch.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      fprintf(stderr, "%s: %s (line %d)\n", #x, cudaGetErrorString(e), __LINE__); \
      exit(1);                                                                  \
    }                                                                           \
  } while (0)

__global__ void nop() {}

int main(int argc, char** argv) {
  const size_t bytes = argc > 1 ? strtoull(argv[1], nullptr, 10) : (48u << 20);
  const int pieces = argc > 2 ? atoi(argv[2]) : 6;
  const int iters = 10;
  char *h_src, *h_dst, *d_src, *d_dst;
  CK(cudaHostAlloc(&h_src, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  CK(cudaHostAlloc(&h_dst, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  CK(cudaMalloc(&d_src, bytes));
  CK(cudaMalloc(&d_dst, bytes));
  cudaStream_t s0, s1;
  CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  cudaEvent_t a, b, j;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaEventCreateWithFlags(&j, cudaEventDisableTiming));
  const size_t pb = bytes / pieces;

  auto time_it = [&](const char* name, size_t moved, auto&& body) {
    for (int w = 0; w < 2; ++w) body();
    CK(cudaStreamSynchronize(s0));
    CK(cudaStreamSynchronize(s1));
    CK(cudaEventRecord(a, s0));
    for (int i = 0; i < iters; ++i) body();
    CK(cudaEventRecord(b, s0));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    ms /= iters;
    printf("{\"probe\": \"%s\", \"bytes\": %zu, \"pieces\": %d, \"ms\": %.4f, \"gbs\": %.2f}\n", name,
           moved, pieces, ms, moved / ms / 1e6);
    fflush(stdout);
  };
  auto h2d = [&](cudaStream_t s) {
    for (int p = 0; p < pieces; ++p)
      CK(cudaMemcpyAsync(d_dst + p * pb, h_src + p * pb, pb, cudaMemcpyHostToDevice, s));
  };
  auto d2h = [&](cudaStream_t s) {
    for (int p = 0; p < pieces; ++p)
      CK(cudaMemcpyAsync(h_dst + p * pb, d_src + p * pb, pb, cudaMemcpyDeviceToHost, s));
  };
  time_it("h2d_one_stream", bytes, [&] { h2d(s0); });
  time_it("d2h_one_stream", bytes, [&] { d2h(s0); });
  time_it("h2d_then_d2h_one_stream", 2 * bytes, [&] { h2d(s0); d2h(s0); });
  time_it("h2d_d2h_two_streams", 2 * bytes, [&] {
    CK(cudaEventRecord(j, s0));
    CK(cudaStreamWaitEvent(s1, j, 0));
    d2h(s1);
    h2d(s0);
    CK(cudaEventRecord(j, s1));
    CK(cudaStreamWaitEvent(s0, j, 0));
  });
  for (unsigned flags : {0u, (unsigned)cudaMemcpyFlagPreferOverlapWithCompute}) {
    std::vector<void*> dsts, srcs;
    std::vector<size_t> sizes;
    for (int p = 0; p < pieces; ++p) {  // interleave the directions
      dsts.push_back(d_dst + p * pb);
      srcs.push_back(h_src + p * pb);
      sizes.push_back(pb);
      dsts.push_back(h_dst + p * pb);
      srcs.push_back(d_src + p * pb);
      sizes.push_back(pb);
    }
    cudaMemcpyAttributes at{};
    at.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
    at.flags = flags;
    size_t idx = 0, fail = 0;
    time_it(flags ? "batch_h2d_d2h_prefer_overlap" : "batch_h2d_d2h", 2 * bytes, [&] {
      CK(cudaMemcpyBatchAsync(dsts.data(), srcs.data(), sizes.data(), dsts.size(), &at, &idx, 1,
                              &fail, s0));
    });
    std::vector<void*> d1(dsts.begin(), dsts.begin() + 1), s1v(srcs.begin(), srcs.begin() + 1);
    time_it(flags ? "batch_h2d_only_prefer_overlap" : "batch_h2d_only", bytes, [&] {
      std::vector<void*> dd, ss;
      std::vector<size_t> zz;
      for (int p = 0; p < pieces; ++p) {
        dd.push_back(d_dst + p * pb);
        ss.push_back(h_src + p * pb);
        zz.push_back(pb);
      }
      CK(cudaMemcpyBatchAsync(dd.data(), ss.data(), zz.data(), dd.size(), &at, &idx, 1, &fail, s0));
    });
  }
  // 2D copies, both directions on two streams vs one stream (the stage/gather shape)
  time_it("memcpy2d_h2d_d2h_one_stream", 2 * bytes, [&] {
    CK(cudaMemcpy2DAsync(d_dst, pb, h_src, pb, pb, pieces, cudaMemcpyHostToDevice, s0));
    CK(cudaMemcpy2DAsync(h_dst, pb, d_src, pb, pb, pieces, cudaMemcpyDeviceToHost, s0));
  });
  return 0;
}

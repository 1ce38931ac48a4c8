// Box probe for the host-link roofline.
// Measures: copy-engine H2D/D2H/bidir over pinned memory, zero-copy SM
// read/write bandwidth over cudaHostRegister'd POSIX SHM, stream mem-op
// support, cross-process stream-wait handshake latency, and concurrent
// zero-copy bandwidth from several processes sharing one GPU (time-slicing).
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_hostlink \
//      tools/probe_hostlink.cu -L/usr/local/cuda/lib64/stubs -lcuda -lpthread
#include <cuda.h>
#include <cuda_runtime.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <string>
#include <thread>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); exit(1);} } while (0)
#define CKD(x) do { CUresult e = (x); if (e != CUDA_SUCCESS) { const char* s; cuGetErrorString(e, &s); \
  fprintf(stderr, "%s:%d %s -> %s\n", __FILE__, __LINE__, #x, s); exit(1);} } while (0)

static double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

__global__ void zc_read(const float4* __restrict__ src, float4* __restrict__ dst, size_t n4) {
  float4 acc = make_float4(0, 0, 0, 0);
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  constexpr int U = 8;
  for (; i + (U - 1) * stride < n4; i += U * stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = src[i + u * stride];
#pragma unroll
    for (int u = 0; u < U; ++u) { acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w; }
  }
  for (; i < n4; i += stride) { float4 v = src[i]; acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w; }
  if (acc.x == 1234.5f) dst[0] = acc;
}

__global__ void zc_copy(const float4* __restrict__ src, float4* __restrict__ dst, size_t n4) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  constexpr int U = 8;
  for (; i + (U - 1) * stride < n4; i += U * stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = src[i + u * stride];
#pragma unroll
    for (int u = 0; u < U; ++u) dst[i + u * stride] = v[u];
  }
  for (; i < n4; i += stride) dst[i] = src[i];
}

static void* shm_map(const char* name, size_t bytes, bool create) {
  int fd = shm_open(name, create ? (O_CREAT | O_RDWR) : O_RDWR, 0600);
  if (fd < 0) { perror("shm_open"); exit(1); }
  if (create && ftruncate(fd, bytes) != 0) { perror("ftruncate"); exit(1); }
  void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) { perror("mmap"); exit(1); }
  return p;
}

static float time_kernel(cudaStream_t s, int iters, const std::function<void()>& f) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  f(); CK(cudaStreamSynchronize(s));
  float best = 1e30f;
  for (int k = 0; k < iters; ++k) {
    CK(cudaEventRecord(a, s)); f(); CK(cudaEventRecord(b, s)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms;
  }
  return best;
}

static void mode_info() {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  char bus[64]; CK(cudaDeviceGetPCIBusId(bus, sizeof bus, dev));
  CUdevice cd; CKD(cuDeviceGet(&cd, dev));
  auto attr = [&](CUdevice_attribute a) { int v = -1; cuDeviceGetAttribute(&v, a, cd); return v; };
  printf("{\"name\":\"%s\",\"sms\":%d,\"bus\":\"%s\",\"pci_domain\":%d,\"gen_mem_gb\":%.1f,"
         "\"can_map_host\":%d,\"pageable_access\":%d,\"host_native_atomic\":%d,"
         "\"stream_memops_v1\":%d,\"memops64\":%d,\"wait_nor\":%d,\"flush_remote\":%d,"
         "\"concurrent_managed\":%d,\"unified_addr\":%d,\"l2_mb\":%.1f}\n",
         p.name, p.multiProcessorCount, bus, p.pciDomainID, p.totalGlobalMem / 1e9,
         p.canMapHostMemory, p.pageableMemoryAccess,
         attr(CU_DEVICE_ATTRIBUTE_HOST_NATIVE_ATOMIC_SUPPORTED),
         attr(CU_DEVICE_ATTRIBUTE_CAN_USE_STREAM_MEM_OPS_V1),
         attr(CU_DEVICE_ATTRIBUTE_CAN_USE_64_BIT_STREAM_MEM_OPS),
         attr(CU_DEVICE_ATTRIBUTE_CAN_USE_STREAM_WAIT_VALUE_NOR),
         attr(CU_DEVICE_ATTRIBUTE_CAN_FLUSH_REMOTE_WRITES),
         p.concurrentManagedAccess, p.unifiedAddressing, p.l2CacheSize / 1048576.0);
}

static void mode_bw() {
  CK(cudaSetDevice(0));
  const size_t bytes = 512ull << 20;
  const size_t n4 = bytes / 16;
  void *h = nullptr, *d = nullptr, *d2 = nullptr, *h2 = nullptr;
  CK(cudaMallocHost(&h, bytes)); CK(cudaMallocHost(&h2, bytes));
  CK(cudaMalloc(&d, bytes)); CK(cudaMalloc(&d2, bytes));
  memset(h, 1, bytes); memset(h2, 1, bytes);
  CK(cudaMemset(d, 0, bytes)); CK(cudaMemset(d2, 0, bytes));
  cudaStream_t s, s2; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  float t;
  t = time_kernel(s, 5, [&] { CK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s)); });
  printf("{\"test\":\"ce_h2d\",\"bytes\":%zu,\"ms\":%.3f,\"gbs\":%.2f}\n", bytes, t, bytes / t / 1e6);
  t = time_kernel(s, 5, [&] { CK(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s)); });
  printf("{\"test\":\"ce_d2h\",\"bytes\":%zu,\"ms\":%.3f,\"gbs\":%.2f}\n", bytes, t, bytes / t / 1e6);
  {
    cudaEvent_t e0, e1, j; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1)); CK(cudaEventCreate(&j));
    float best = 1e30f;
    for (int k = 0; k < 5; ++k) {
      CK(cudaEventRecord(e0, s)); CK(cudaStreamWaitEvent(s2, e0));
      CK(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(h2, d2, bytes, cudaMemcpyDeviceToHost, s2));
      CK(cudaEventRecord(j, s2)); CK(cudaStreamWaitEvent(s, j)); CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1)); float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
    }
    printf("{\"test\":\"ce_bidir\",\"bytes_each\":%zu,\"ms\":%.3f,\"gbs_total\":%.2f}\n", bytes, best, 2 * bytes / best / 1e6);
  }
  // POSIX SHM + cudaHostRegister(mapped|portable): zero-copy SM traffic.
  const char* name = "/fmx-probe-bw";
  shm_unlink(name);
  void* sh = shm_map(name, bytes, true);
  memset(sh, 1, bytes);
  double t0 = now_s();
  CK(cudaHostRegister(sh, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable));
  double treg = now_s() - t0;
  void* shd; CK(cudaHostGetDevicePointer(&shd, sh, 0));
  printf("{\"test\":\"host_register\",\"bytes\":%zu,\"s\":%.3f}\n", bytes, treg);
  t = time_kernel(s, 5, [&] { CK(cudaMemcpyAsync(d, sh, bytes, cudaMemcpyHostToDevice, s)); });
  printf("{\"test\":\"ce_h2d_shm\",\"gbs\":%.2f}\n", bytes / t / 1e6);
  t = time_kernel(s, 5, [&] { CK(cudaMemcpyAsync(sh, d, bytes, cudaMemcpyDeviceToHost, s)); });
  printf("{\"test\":\"ce_d2h_shm\",\"gbs\":%.2f}\n", bytes / t / 1e6);
  int grids[] = {8, 16, 24, 32, 48, 64, 148, 296, 592};
  int threads_list[] = {256, 512, 1024};
  for (int th : threads_list)
    for (int g : grids) {
      float tr = time_kernel(s, 3, [&] { zc_read<<<g, th, 0, s>>>((const float4*)shd, (float4*)d, n4); });
      float tw = time_kernel(s, 3, [&] { zc_copy<<<g, th, 0, s>>>((const float4*)d2, (float4*)shd, n4); });
      float tc = time_kernel(s, 3, [&] { zc_copy<<<g, th, 0, s>>>((const float4*)shd, (float4*)d, n4); });
      printf("{\"test\":\"zc\",\"blocks\":%d,\"threads\":%d,\"read_gbs\":%.2f,\"write_gbs\":%.2f,\"h2d_copy_gbs\":%.2f}\n",
             g, th, bytes / tr / 1e6, bytes / tw / 1e6, bytes / tc / 1e6);
    }
  // simultaneous zero-copy read + write (bidirectional, SM driven), two streams
  for (int g : {16, 32, 74, 148}) {
    cudaEvent_t e0, e1, j; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1)); CK(cudaEventCreate(&j));
    float best = 1e30f;
    size_t half = n4 / 2;
    for (int k = 0; k < 4; ++k) {
      CK(cudaEventRecord(e0, s)); CK(cudaStreamWaitEvent(s2, e0));
      zc_copy<<<g, 512, 0, s>>>((const float4*)shd, (float4*)d, half);
      zc_copy<<<g, 512, 0, s2>>>((const float4*)d2, (float4*)shd + half, half);
      CK(cudaEventRecord(j, s2)); CK(cudaStreamWaitEvent(s, j)); CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1)); float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
    }
    printf("{\"test\":\"zc_bidir\",\"blocks_each\":%d,\"gbs_total\":%.2f}\n", g, 2 * half * 16 / best / 1e6);
  }
  CK(cudaHostUnregister(sh));
  munmap(sh, bytes);
  shm_unlink(name);
  // host DRAM bandwidth: multithreaded memcpy
  {
    unsigned nt = std::thread::hardware_concurrency();
    size_t hb = 1ull << 30;
    char* a = (char*)aligned_alloc(4096, hb); char* b = (char*)aligned_alloc(4096, hb);
    memset(a, 1, hb); memset(b, 2, hb);
    for (unsigned use : {1u, nt / 4 ? nt / 4 : 1u, nt / 2 ? nt / 2 : 1u, nt}) {
      double best = 1e30;
      for (int k = 0; k < 3; ++k) {
        std::vector<std::thread> ts; double t0 = now_s();
        for (unsigned i = 0; i < use; ++i) ts.emplace_back([&, i] {
          size_t per = hb / use; memcpy(b + i * per, a + i * per, per); });
        for (auto& x : ts) x.join();
        double dt = now_s() - t0; if (dt < best) best = dt;
      }
      printf("{\"test\":\"host_memcpy\",\"threads\":%u,\"gbs_rw\":%.2f}\n", use, 2.0 * hb / best / 1e9);
    }
  }
}

// Cross-process: two ranks on the same GPU. Role 0 creates the segment.
// (1) stream wait/write handshake round-trip latency; (2) concurrent zero-copy
// read bandwidth while the other rank does the same.
struct Ctl { std::atomic<int> ready[8]; std::atomic<int> go; int pad[16]; unsigned flags[64][16]; };

static void mode_pair(int role, int nproc, int blocks) {
  CK(cudaSetDevice(0));
  CK(cudaFree(0));
  const char* name = "/fmx-probe-pair";
  const size_t data_bytes = 256ull << 20;
  const size_t total = 4096 + data_bytes * nproc;
  if (role == 0) { shm_unlink(name); }
  void* base = nullptr;
  if (role == 0) base = shm_map(name, total, true);
  else { for (int k = 0; k < 10000; ++k) { int fd = shm_open(name, O_RDWR, 0600); if (fd >= 0) { close(fd); break; } usleep(1000);} usleep(200000); base = shm_map(name, total, false); }
  CK(cudaHostRegister(base, total, cudaHostRegisterMapped | cudaHostRegisterPortable));
  char* dbase; CK(cudaHostGetDevicePointer((void**)&dbase, base, 0));
  Ctl* ctl = (Ctl*)base;
  ctl->ready[role].store(1);
  for (int i = 0; i < nproc; ++i) while (ctl->ready[i].load() != 1) usleep(100);
  cudaStream_t s; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  CUstream cs = (CUstream)s;
  CUdeviceptr myflag = (CUdeviceptr)(dbase + offsetof(Ctl, flags) + role * 64);
  CUdeviceptr peerflag = (CUdeviceptr)(dbase + offsetof(Ctl, flags) + ((role + 1) % nproc) * 64);
  // ping-pong ring over nproc ranks
  const int iters = 2000;
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  CK(cudaEventRecord(a, s));
  for (int k = 1; k <= iters; ++k) {
    if (role == 0) {
      CKD(cuStreamWriteValue32(cs, myflag, k, 0));
      CUdeviceptr prev = (CUdeviceptr)(dbase + offsetof(Ctl, flags) + (nproc - 1) * 64);
      CKD(cuStreamWaitValue32(cs, prev, k, CU_STREAM_WAIT_VALUE_GEQ));
    } else {
      CUdeviceptr prev = (CUdeviceptr)(dbase + offsetof(Ctl, flags) + (role - 1) * 64);
      CKD(cuStreamWaitValue32(cs, prev, k, CU_STREAM_WAIT_VALUE_GEQ));
      CKD(cuStreamWriteValue32(cs, myflag, k, 0));
    }
  }
  CK(cudaEventRecord(b, s)); CK(cudaEventSynchronize(b));
  float ms; CK(cudaEventElapsedTime(&ms, a, b));
  (void)peerflag;
  printf("{\"test\":\"ring_memop\",\"role\":%d,\"nproc\":%d,\"us_per_hop\":%.2f}\n", role, nproc, ms * 1000.0 / iters / nproc);
  fflush(stdout);
  // barrier
  ctl->ready[role].store(2);
  for (int i = 0; i < nproc; ++i) while (ctl->ready[i].load() < 2) usleep(100);
  // concurrent zero-copy read of own region
  void* d; CK(cudaMalloc(&d, data_bytes));
  const float4* src = (const float4*)(dbase + 4096 + role * data_bytes);
  size_t n4 = data_bytes / 16;
  zc_read<<<blocks, 512, 0, s>>>(src, (float4*)d, n4); CK(cudaStreamSynchronize(s));
  ctl->ready[role].store(3);
  for (int i = 0; i < nproc; ++i) while (ctl->ready[i].load() < 3) ;
  double t0 = now_s();
  CK(cudaEventRecord(a, s));
  for (int k = 0; k < 5; ++k) zc_read<<<blocks, 512, 0, s>>>(src, (float4*)d, n4);
  CK(cudaEventRecord(b, s)); CK(cudaEventSynchronize(b));
  double wall = now_s() - t0;
  CK(cudaEventElapsedTime(&ms, a, b));
  printf("{\"test\":\"concurrent_zc_read\",\"role\":%d,\"nproc\":%d,\"blocks\":%d,\"event_gbs\":%.2f,\"wall_gbs\":%.2f,\"wall_s\":%.4f,\"t0\":%.6f}\n",
         role, nproc, blocks, 5 * data_bytes / ms / 1e6, 5 * data_bytes / wall / 1e9, wall, t0);
  // concurrent zero-copy write of own region (D2H)
  ctl->ready[role].store(4);
  for (int i = 0; i < nproc; ++i) while (ctl->ready[i].load() < 4) ;
  t0 = now_s();
  CK(cudaEventRecord(a, s));
  for (int k = 0; k < 5; ++k) zc_copy<<<blocks, 512, 0, s>>>((const float4*)d, (float4*)src, n4);
  CK(cudaEventRecord(b, s)); CK(cudaEventSynchronize(b));
  wall = now_s() - t0;
  CK(cudaEventElapsedTime(&ms, a, b));
  printf("{\"test\":\"concurrent_zc_write\",\"role\":%d,\"nproc\":%d,\"blocks\":%d,\"event_gbs\":%.2f,\"wall_gbs\":%.2f,\"wall_s\":%.4f,\"t0\":%.6f}\n",
         role, nproc, blocks, 5 * data_bytes / ms / 1e6, 5 * data_bytes / wall / 1e9, wall, t0);
  ctl->ready[role].store(5);
  for (int i = 0; i < nproc; ++i) while (ctl->ready[i].load() < 5) usleep(100);
  CK(cudaHostUnregister(base));
  if (role == 0) shm_unlink(name);
}


// Two processes, each moving 256 MB per iteration in its own direction/method:
// r = SM zero-copy read (H2D), w = SM zero-copy write (D2H), H = CE H2D, D = CE D2H.
static void mode_dir(int role, int nproc, const char* kinds, int blocks) {
  CK(cudaSetDevice(0)); CK(cudaFree(0));
  const char* name = "/fmx-probe-dir";
  const size_t data_bytes = 256ull << 20;
  const size_t total = 4096 + data_bytes * nproc;
  if (role == 0) shm_unlink(name);
  void* base = nullptr;
  if (role == 0) base = shm_map(name, total, true);
  else { for (int k = 0; k < 10000; ++k) { int fd = shm_open(name, O_RDWR, 0600); if (fd >= 0) { close(fd); break; } usleep(1000);} usleep(200000); base = shm_map(name, total, false); }
  CK(cudaHostRegister(base, total, cudaHostRegisterMapped | cudaHostRegisterPortable));
  char* dbase; CK(cudaHostGetDevicePointer((void**)&dbase, base, 0));
  Ctl* ctl = (Ctl*)base;
  cudaStream_t s; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  void* d; CK(cudaMalloc(&d, data_bytes));
  char* hreg = (char*)base + 4096 + role * data_bytes;
  char* dreg = dbase + 4096 + role * data_bytes;
  size_t n4 = data_bytes / 16;
  char k = kinds[role];
  auto run = [&] {
    if (k == 'r') zc_read<<<blocks, 512, 0, s>>>((const float4*)dreg, (float4*)d, n4);
    else if (k == 'w') zc_copy<<<blocks, 512, 0, s>>>((const float4*)d, (float4*)dreg, n4);
    else if (k == 'H') CK(cudaMemcpyAsync(d, hreg, data_bytes, cudaMemcpyHostToDevice, s));
    else if (k == 'D') CK(cudaMemcpyAsync(hreg, d, data_bytes, cudaMemcpyDeviceToHost, s));
  };
  run(); CK(cudaStreamSynchronize(s));
  ctl->ready[role].store(1);
  for (int i = 0; i < nproc; ++i) while (ctl->ready[i].load() < 1) ;
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  double t0 = now_s();
  CK(cudaEventRecord(a, s));
  for (int it = 0; it < 10; ++it) run();
  CK(cudaEventRecord(b, s)); CK(cudaEventSynchronize(b));
  double wall = now_s() - t0; float ms; CK(cudaEventElapsedTime(&ms, a, b));
  printf("{\"test\":\"dir\",\"kinds\":\"%s\",\"role\":%d,\"kind\":\"%c\",\"blocks\":%d,\"event_gbs\":%.2f,\"wall_gbs\":%.2f,\"t0\":%.6f,\"t1\":%.6f}\n",
         kinds, role, k, blocks, 10 * data_bytes / ms / 1e6, 10 * data_bytes / wall / 1e9, t0, t0 + wall);
  ctl->ready[role].store(2);
  for (int i = 0; i < nproc; ++i) while (ctl->ready[i].load() < 2) usleep(100);
  CK(cudaHostUnregister(base));
  if (role == 0) shm_unlink(name);
}

int main(int argc, char** argv) {
  std::string m = argc > 1 ? argv[1] : "info";
  CKD(cuInit(0));
  if (m == "info") mode_info();
  else if (m == "bw") mode_bw();
  else if (m == "dir") mode_dir(atoi(argv[2]), atoi(argv[3]), argv[4], argc > 5 ? atoi(argv[5]) : 16);
  else if (m == "pair") mode_pair(atoi(argv[2]), atoi(argv[3]), argc > 4 ? atoi(argv[4]) : 16);
  return 0;
}

// sm_100a kernels of the SHM data path.
//
//   fmx_copy_kernel    - batched segment copy (stage: HBM -> SHM with 128-bit
//                        stores; gather / broadcast: SHM -> HBM with 128-bit
//                        cache-volatile loads).  One blockIdx.y per segment.
//   fmx_reduce_kernel  - owner-chunk reduction: n sources (peer slots in SHM or
//                        HBM scratch, own chunk in HBM), fixed ascending-rank
//                        fp32 sum (__fadd_rn, no contraction), fused
//                        pre-multiply (DDP mean) / pre-divide / post-scale
//                        and bf16 RNE cast, written to
//                        the rank's HBM result and its SHM result slot.
//
// All host-link traffic is streaming (each byte touched once), so the kernels
// are memory-level-parallelism bound: 128-bit accesses, several independent
// vectors in flight per thread, grid-stride over the piece.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "../../include/flexshm.h"
#include "fmx_args.h"

namespace fmx {

constexpr int kMaxSegs = 64;

struct CopySeg {
  const char* src;
  char* dst;
  size_t bytes;
};

struct CopyArgs {
  CopySeg seg[kMaxSegs];
  int nseg;
  int src_sys;           // 1: sources live in mapped host memory -> ld.cv
  uint32_t* flag;        // non-null: the last CTA to finish releases *flag = flag_value
  uint32_t flag_value;   //   (system scope, after every CTA's stores) - a fused signal
  unsigned int* ctas_done;  // device counter for the last-CTA election (reset by the winner)
};

// Fused signal: every CTA fences its stores at system scope and counts itself
// done; the last one resets the counter and releases the flag, so a peer
// that sees the flag (stream wait on host memory) sees every byte copied.
__device__ __forceinline__ void release_flag_when_grid_done(const CopyArgs& a) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const unsigned int total = gridDim.x * gridDim.y;
    if (atomicAdd(a.ctas_done, 1u) == total - 1) {
      *a.ctas_done = 0;
      __threadfence_system();
      asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.flag), "r"(a.flag_value)
                   : "memory");
    }
  }
}


__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Fused flag wait (ReduceArgs::wait_flags): thread q of the CTA polls rank q's
// flag with acquire loads at system scope; the CTA barrier then orders every
// thread's source loads after the peers' releases.  Only for MPS-concurrent
// ranks (the caller checks): a spinning CTA must not hold a time slice.
__device__ __forceinline__ void wait_flags_cta(const char* base, size_t stride, int n, int skip,
                                               uint32_t v) {
  for (int q = threadIdx.x; q < n; q += blockDim.x) {
    if (q == skip) continue;
    const uint32_t* f = (const uint32_t*)(base + (size_t)q * stride);
    while ((int32_t)(ld_acquire_sys(f) - v) < 0) __nanosleep(64);
  }
  __syncthreads();
}

__device__ __forceinline__ uint4 ld_cv_v4(const void* p) {
  uint4 v;
  asm volatile("ld.global.cv.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ uint4 ld_v4(const void* p) {
  uint4 v;
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void st_v4(void* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// ---------------------------------------------------------------- copy

template <int U>
__global__ void __launch_bounds__(512) fmx_copy_kernel(const __grid_constant__ CopyArgs a) {
  const CopySeg s = a.seg[blockIdx.y];
  const size_t nvec = s.bytes / 16;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if ((((uintptr_t)s.src | (uintptr_t)s.dst) & 15) == 0) {
    for (; i + (U - 1) * stride < nvec; i += U * stride) {
      uint4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
        v[u] = a.src_sys ? ld_cv_v4(s.src + (i + u * stride) * 16)
                         : ld_v4(s.src + (i + u * stride) * 16);
#pragma unroll
      for (int u = 0; u < U; ++u) st_v4(s.dst + (i + u * stride) * 16, v[u]);
    }
    for (; i < nvec; i += stride)
      st_v4(s.dst + i * 16, a.src_sys ? ld_cv_v4(s.src + i * 16) : ld_v4(s.src + i * 16));
    // byte tail
    size_t t = nvec * 16 + (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; t < s.bytes; t += stride) s.dst[t] = ((volatile const char*)s.src)[t];
  } else {
    for (; i < s.bytes; i += stride) s.dst[i] = ((volatile const char*)s.src)[i];
  }
  if (a.flag) release_flag_when_grid_done(a);
}

// ---------------------------------------------------------------- reduce

template <typename T>
struct Elem;

template <>
struct Elem<float> {
  static constexpr int kVec = 4;
  __device__ static __forceinline__ void widen(const uint4& v, float* f) {
    f[0] = __uint_as_float(v.x);
    f[1] = __uint_as_float(v.y);
    f[2] = __uint_as_float(v.z);
    f[3] = __uint_as_float(v.w);
  }
  __device__ static __forceinline__ uint4 narrow(const float* f) {
    return make_uint4(__float_as_uint(f[0]), __float_as_uint(f[1]), __float_as_uint(f[2]),
                      __float_as_uint(f[3]));
  }
  __device__ static __forceinline__ float prediv(float x, float d) { return __fdiv_rn(x, d); }
  __device__ static __forceinline__ float premul(float x, float m) { return __fmul_rn(x, m); }
  __device__ static __forceinline__ float load1(const char* p) {
    return *(volatile const float*)p;
  }
  __device__ static __forceinline__ void store1(char* p, float v) { *(float*)p = v; }
};

__device__ __forceinline__ float bf16_bits_to_f32(uint32_t b) { return __uint_as_float(b << 16); }
__device__ __forceinline__ uint32_t f32_to_bf16_bits(float f) {
  return (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(f));
}

template <>
struct Elem<__nv_bfloat16> {
  static constexpr int kVec = 8;
  __device__ static __forceinline__ void widen(const uint4& v, float* f) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      f[2 * k] = bf16_bits_to_f32(w[k] & 0xFFFFu);
      f[2 * k + 1] = bf16_bits_to_f32(w[k] >> 16);
    }
  }
  __device__ static __forceinline__ uint4 narrow(const float* f) {
    uint32_t w[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) w[k] = f32_to_bf16_bits(f[2 * k]) | (f32_to_bf16_bits(f[2 * k + 1]) << 16);
    return make_uint4(w[0], w[1], w[2], w[3]);
  }
  // A bf16 bucket divided in place is rounded back to bf16 before the sum.
  __device__ static __forceinline__ float prediv(float x, float d) {
    return bf16_bits_to_f32(f32_to_bf16_bits(__fdiv_rn(x, d)));
  }
  // ATen's bf16 `mul by an fp32 scalar`: fp32 product, rounded to bf16
  __device__ static __forceinline__ float premul(float x, float m) {
    return bf16_bits_to_f32(f32_to_bf16_bits(__fmul_rn(x, m)));
  }
  __device__ static __forceinline__ float load1(const char* p) {
    return bf16_bits_to_f32(*(volatile const unsigned short*)p);
  }
  __device__ static __forceinline__ void store1(char* p, float v) {
    *(unsigned short*)p = (unsigned short)f32_to_bf16_bits(v);
  }
};

// One rank's contribution under the op's input scaling (PREDIV / PREMUL);
// OP is a template parameter so each op compiles to its own straight-line
// code (no division path in the DDP-mean kernel, no spills).
template <typename T, int OP>
__device__ __forceinline__ float scale_in(float x, float f) {
  if constexpr (OP == FMX_OP_PREMUL_SUM) return Elem<T>::premul(x, f);
  else if constexpr (OP == FMX_OP_PREDIV_SUM) return Elem<T>::prediv(x, f);
  else return x;
}

template <int OP>
__device__ __forceinline__ float scale_out(float acc, float f) {
  if constexpr (OP == FMX_OP_SUM_POSTSCALE) return __fmul_rn(acc, f);
  else return acc;
}

// Sum of the vector positions i + u * stride, u in [U0, U0 + G), across all
// sources, rank order; the loads of all G positions of a source batch are
// issued before any is consumed (G x B independent 128-bit loads in flight).
template <typename T, int OP, int U, int U0, int G>
__device__ __forceinline__ void reduce_group(const ReduceArgs& a, size_t i, size_t stride, size_t nvec,
                                             float (&acc)[U][Elem<T>::kVec]) {
  using E = Elem<T>;
  constexpr int V = E::kVec;
  constexpr int B = 8;  // sources loaded per batch
  for (int q0 = 0; q0 < a.nsrc; q0 += B) {
    uint4 raw[G][B];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int u = U0 + g;
      if (i + u * stride >= nvec) continue;
      const size_t off = (i + u * stride) * 16;
#pragma unroll
      for (int b = 0; b < B; ++b) {
        const int q = q0 + b;
        if (q < a.nsrc)
          raw[g][b] = ((a.sys_mask >> q) & 1) ? ld_cv_v4(a.src[q] + off) : ld_v4(a.src[q] + off);
      }
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int u = U0 + g;
      if (i + u * stride >= nvec) continue;
#pragma unroll
      for (int b = 0; b < B; ++b) {
        const int q = q0 + b;
        if (q < a.nsrc) {
          float x[V];
          E::widen(raw[g][b], x);
#pragma unroll
          for (int k = 0; k < V; ++k) {
            const float c = scale_in<T, OP>(x[k], a.factor);
            acc[u][k] = q == 0 ? c : __fadd_rn(acc[u][k], c);
          }
        }
      }
    }
  }
}

// One vector position's sources, rank order (host sources: one vector's
// sources in flight at a time).
template <typename T, int OP>
__device__ __forceinline__ void reduce_one(const ReduceArgs& a, size_t off, float* acc) {
  using E = Elem<T>;
  constexpr int V = E::kVec;
  constexpr int B = 8;  // sources loaded per batch
  for (int q0 = 0; q0 < a.nsrc; q0 += B) {
    uint4 raw[B];
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int q = q0 + b;
      if (q < a.nsrc)
        raw[b] = ((a.sys_mask >> q) & 1) ? ld_cv_v4(a.src[q] + off) : ld_v4(a.src[q] + off);
    }
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const int q = q0 + b;
      if (q < a.nsrc) {
        float x[V];
        E::widen(raw[b], x);
#pragma unroll
        for (int k = 0; k < V; ++k) {
          const float c = scale_in<T, OP>(x[k], a.factor);
          acc[k] = q == 0 ? c : __fadd_rn(acc[k], c);
        }
      }
    }
  }
}

// Sum of U vector positions (i, i + stride, ...) across all sources, rank
// order.  HBM sources (the copy-engine transport): the loads of all U
// positions are in flight together - inside a 1g-sized partition the kernel
// is latency bound, and one round trip per U vectors instead of per vector
// cuts the HBM-only launch (result slot by copy engine) 78.5 -> 62-67 us
// (r02/r5b).  Host sources (zero-copy transport, one-shot): one position's
// sources at a time, the round-1 form and register count (70) - 14 concurrent
// host reads per thread made the 64 KiB one-shot at 7 ranks 5-11 % slower
// (r02/r5e, r5f).  The per-element arithmetic and its order are the same.
template <typename T, int OP, int U, bool HOST_SRC>
__device__ __forceinline__ void reduce_vecs(const ReduceArgs& a, size_t i, size_t stride, size_t nvec,
                                            float (&acc)[U][Elem<T>::kVec]) {
  if constexpr (HOST_SRC) {
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i + u * stride < nvec) reduce_one<T, OP>(a, (i + u * stride) * 16, acc[u]);
  } else
    reduce_group<T, OP, U, 0, U>(a, i, stride, nvec, acc);
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int k = 0; k < Elem<T>::kVec; ++k) acc[u][k] = scale_out<OP>(acc[u][k], a.factor);
}

// The fused SGD step of one element (ReduceArgs::sgd): torch's multi-tensor SGD
// (torch/optim/sgd.py _multi_tensor_sgd) op by op - _foreach_add with alpha is
// `a + alpha * b` contracted to one FMA, _foreach_mul one rounded product - so
// the owner's update is bit-identical to every rank updating its replica.
// `p` is the old parameter; returns the new one and updates *m.
__device__ __forceinline__ float sgd_step(const ReduceArgs& a, float g, float p, float* m) {
  if (a.wd != 0.f) g = __fmaf_rn(a.wd, p, g);
  float d = g;
  if (a.mu != 0.f) {
    *m = a.init ? g : __fmaf_rn(1.f - a.damp, g, __fmul_rn(*m, a.mu));
    d = a.nesterov ? __fmaf_rn(a.mu, *m, g) : *m;
  }
  return __fmaf_rn(-a.lr, d, p);
}

// One element (tails and the unaligned path).
template <typename T, int OP, bool SGD = false>
__device__ __forceinline__ void reduce_elem(const ReduceArgs& a, size_t e) {
  using E = Elem<T>;
  const size_t esz = sizeof(T);
  float acc = 0.f;
  for (int q = 0; q < a.nsrc; ++q) {
    const float c = scale_in<T, OP>(E::load1(a.src[q] + e * esz), a.factor);
    acc = q == 0 ? c : __fadd_rn(acc, c);
  }
  acc = scale_out<OP>(acc, a.factor);
  if constexpr (SGD) {
    float m = a.mom ? ((const float*)a.mom)[e] : 0.f;
    acc = sgd_step(a, acc, E::load1(a.out_dev + e * esz), &m);
    if (a.mom) ((float*)a.mom)[e] = m;
  }
  E::store1(a.out_dev + e * esz, acc);
  for (int k = 1; k < a.n_rep; ++k) E::store1(a.out_dev + k * a.rep_stride + e * esz, acc);
  if (a.out_sys) E::store1(a.out_sys + e * esz, acc);
}

template <typename T, int U, int OP, bool SGD = false, bool HOST_SRC = false>
__global__ void __launch_bounds__(256, 2) fmx_reduce_kernel(const __grid_constant__ ReduceArgs a) {
  using E = Elem<T>;
  constexpr int V = E::kVec;
  if (a.wait_flags) wait_flags_cta(a.wait_flags, a.wait_stride, a.nsrc, a.wait_skip, a.wait_value);
  const size_t nvec = a.len / V;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (size_t i = tid; i < nvec; i += U * stride) {
    float acc[U][V];
    reduce_vecs<T, OP, U, HOST_SRC>(a, i, stride, nvec, acc);
    if constexpr (SGD) {   // fp32 only: V = 4 parameters and momenta per vector
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (i + u * stride >= nvec) continue;
        const size_t off = (i + u * stride) * 16;
        float p[V], m[V] = {};
        E::widen(ld_v4(a.out_dev + off), p);
        if (a.mom) E::widen(ld_v4(a.mom + off), m);
#pragma unroll
        for (int k = 0; k < V; ++k) acc[u][k] = sgd_step(a, acc[u][k], p[k], &m[k]);
        if (a.mom) st_v4(a.mom + off, E::narrow(m));
      }
    }
    uint4 o[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (i + u * stride < nvec) {
        o[u] = E::narrow(acc[u]);
        st_v4(a.out_dev + (i + u * stride) * 16, o[u]);
        if (a.out_sys) st_v4(a.out_sys + (i + u * stride) * 16, o[u]);
      }
    }
    // host path: the same result into every replica (one per destination region)
    for (int k = 1; k < a.n_rep; ++k) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (i + u * stride < nvec) st_v4(a.out_dev + k * a.rep_stride + (i + u * stride) * 16, o[u]);
    }
  }
  // element tail (len not a multiple of the vector width)
  for (size_t e = nvec * V + tid; e < a.len; e += stride) reduce_elem<T, OP, SGD>(a, e);
}

// Unaligned fallback: one element per thread iteration.
template <typename T, int OP, bool SGD = false>
__global__ void __launch_bounds__(256) fmx_reduce_scalar_kernel(const __grid_constant__ ReduceArgs a) {
  if (a.wait_flags) wait_flags_cta(a.wait_flags, a.wait_stride, a.nsrc, a.wait_skip, a.wait_value);
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < a.len; e += stride)
    reduce_elem<T, OP, SGD>(a, e);
}

// Host-side dispatch over (dtype, op, alignment): grid capped at 8 x 148 CTAs
// of 256 threads, 2 vectors per thread in flight.
constexpr int kReduceThreads = 256, kReduceU = 2, kReduceGridCap = 1184;

template <typename T, int OP, bool SGD = false>
inline void launch_reduce_t(const ReduceArgs& a, bool aligned, cudaStream_t s, int cap) {
  constexpr int V = Elem<T>::kVec;
  auto grid = [cap](size_t items) {
    size_t g = (items + kReduceThreads - 1) / kReduceThreads;
    return (int)(g < 1 ? 1 : g > (size_t)cap ? cap : g);
  };
  const int g = grid((a.len / V + kReduceU - 1) / kReduceU + 1);
  if (aligned && a.sys_mask)   // sources in mapped host memory (zero-copy, one-shot)
    fmx_reduce_kernel<T, kReduceU, OP, SGD, true><<<g, kReduceThreads, 0, s>>>(a);
  else if (aligned)
    fmx_reduce_kernel<T, kReduceU, OP, SGD, false><<<g, kReduceThreads, 0, s>>>(a);
  else
    fmx_reduce_scalar_kernel<T, OP, SGD><<<grid(a.len), kReduceThreads, 0, s>>>(a);
}

template <typename T>
inline void launch_reduce_op(const ReduceArgs& a, bool aligned, cudaStream_t s, int cap) {
  if constexpr (std::is_same<T, float>::value) {
    if (a.sgd) {   // fused SGD step: DDP's mean (PREMUL) or a plain sum
      if (a.op == FMX_OP_PREMUL_SUM) return launch_reduce_t<T, FMX_OP_PREMUL_SUM, true>(a, aligned, s, cap);
      return launch_reduce_t<T, FMX_OP_SUM, true>(a, aligned, s, cap);
    }
  }
  switch (a.op) {
    case FMX_OP_SUM_POSTSCALE: return launch_reduce_t<T, FMX_OP_SUM_POSTSCALE>(a, aligned, s, cap);
    case FMX_OP_PREDIV_SUM: return launch_reduce_t<T, FMX_OP_PREDIV_SUM>(a, aligned, s, cap);
    case FMX_OP_PREMUL_SUM: return launch_reduce_t<T, FMX_OP_PREMUL_SUM>(a, aligned, s, cap);
    default: return launch_reduce_t<T, FMX_OP_SUM>(a, aligned, s, cap);
  }
}

// cap: most CTAs per launch (kReduceGridCap; FMX_REDUCE_CTAS lowers it per communicator)
inline void launch_reduce(const ReduceArgs& a, int dtype, bool aligned, cudaStream_t s,
                          int cap = kReduceGridCap) {
  if (dtype == FMX_FLOAT32)
    launch_reduce_op<float>(a, aligned, s, cap);
  else
    launch_reduce_op<__nv_bfloat16>(a, aligned, s, cap);
}

// ---------------------------------------------------------------- stamps

// Pipeline timeline probe (fmx_comm_set_stamps): one thread writes the GPU's
// global nanosecond timer - the same clock for every process on the GPU - and
// a (lane, op, info) tag into the next entry of a device buffer, so stamps
// enqueued after each operation of every rank line up on one time axis.

__global__ void fmx_nop_kernel() {}

__global__ void fmx_stamp_kernel(Stamp* slot, uint32_t tag, uint32_t info) {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  slot->t_ns = t;
  slot->tag = tag;
  slot->info = info;
}

}  // namespace fmx

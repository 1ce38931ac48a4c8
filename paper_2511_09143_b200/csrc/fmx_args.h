// Argument blocks shared by the host schedule and the sm_100a kernels
// (plain C++: no CUDA headers, so the schedule compiles with g++).
#pragma once

#include <stddef.h>
#include <stdint.h>

#include "../../include/flexshm.h"

namespace fmx {

struct ReduceArgs {
  const char* src[FMX_MAX_RANKS];  // rank-ordered sources
  uint64_t sys_mask;               // bit q set: src[q] is mapped host memory
  char* out_dev;                   // HBM result (may alias src[own])
  char* out_sys;                   // SHM result slot (may be null)
  size_t rep_stride;               // n_rep > 1: also write the result at out_dev + k*rep_stride
  int n_rep;                       // (host path: one replica per destination region)
  size_t len;                      // elements
  int nsrc;
  int op;
  float factor;
  // non-null: before reading any source, every CTA waits until the flag of
  // each rank q != wait_skip (at wait_flags + q * wait_stride) is cyclically
  // >= wait_value - the one-shot's OS_READY wait fused into its reduction
  const char* wait_flags;
  size_t wait_stride;
  uint32_t wait_value;
  int wait_skip;
  // fused SGD epilogue (fmx_allreduce_sgd; fp32): the reduced gradient g of
  // element e updates the parameter p = out_dev[e] in place and its momentum
  // mom[e], torch's multi-tensor SGD step op by op, and p (not g) is what
  // goes to out_sys and the all-gather:
  //   g = wd ? g + wd*p : g;  m = init ? g : m*mu + (1-damp)*g;
  //   d = nesterov ? g + mu*m : m;  p = p + (-lr)*d     (x + a*y as one FMA)
  int sgd;        // 1: apply the epilogue
  char* mom;      // momentum of the elements of out_dev (null: momentum 0)
  float lr, mu, damp, wd;
  int nesterov, init;
};

// Pipeline timeline probe entry (fmx_comm_set_stamps).
struct Stamp {
  uint64_t t_ns;
  uint32_t tag;   // lane << 8 | op kind
  uint32_t info;  // flag value / bytes / event id
};

}  // namespace fmx

// Communicator, SHM segment manager and the chunk pipeline of libflexshm.
//
// Design:
//  * One POSIX SHM segment per communicator, "/fmx-<job_key>", created by rank
//    0, pinned + device-mapped by every rank (cudaHostRegister Mapped |
//    Portable).  MIG forbids cross-instance P2P/NVLink (reference
//    PAPER.md:262), so host memory is the only shared medium - the same
//    transport NCCL's SHM path gives the paper's ranks.
//  * Bootstrap = the paper's patched ncclCommInitRank:
//    every rank publishes its fmx_peer_info into the segment's peer table,
//    then every rank applies discover_peers / build_topology rules
//    (flexshm_host.cpp) to the full table, so all ranks agree on failure.
//  * Allreduce = reduce-scatter + all-gather through the segment.  Rank r owns
//    chunk r of the flat buffer (16-byte aligned chunk boundaries).  Each
//    chunk is pipelined in rounds of `slice` elements; round R uses slot
//    R % K of every region (K = 2 by default).  Per round a rank (1) stages
//    its pieces of the other owners' chunks into in-slot[owner][r], (2) after
//    every peer signalled STAGED, reduces its own chunk in ascending rank
//    order (own contribution read from HBM at its own rank position) into
//    its HBM result and out-slot[r], (3) after every peer signalled REDUCED,
//    gathers the other owners' results.
//  * Flags are monotone 32-bit round counters in the segment, one 64-byte
//    line each, written with cuStreamWriteValue-class stream memory ops
//    (system-scope fence before the write) and waited on with stream
//    memory-op waits.  No SM ever spins: a wait parks the stream in the GPU
//    front end, which matters because rank processes sharing one GPU without
//    MPS are time-sliced.  Slot reuse needs no credit messages: events on the
//    lanes carry "every peer is past round R-K".
//  * The schedule itself (plans, trace for the model checker) lives in
//    flexshm_plan.cpp; this file holds the CUDA half: CudaSink, the lanes,
//    the segment, and the C API.
#include <cuda.h>
#include <cuda_runtime.h>
#include <errno.h>
#include <fcntl.h>
#include <signal.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "fmx_comm.h"
#include "flexshm_kernels.cuh"

using namespace fmx;

namespace {

typedef CUresult (*PFN_batchMemOp)(CUstream, unsigned int, CUstreamBatchMemOpParams*,
                                   unsigned int);
typedef CUresult (*PFN_streamGetCtx)(CUstream, CUcontext*);
typedef CUresult (*PFN_ctxPush)(CUcontext);
typedef CUresult (*PFN_ctxPop)(CUcontext*);
typedef CUresult (*PFN_ctxGetCurrent)(CUcontext*);
PFN_batchMemOp g_batch = nullptr;
PFN_ctxGetCurrent g_ctx_current = nullptr;
PFN_streamGetCtx g_stream_ctx = nullptr;
PFN_ctxPush g_ctx_push = nullptr;
PFN_ctxPop g_ctx_pop = nullptr;
std::once_flag g_driver_once;
int g_driver_status = FMX_OK;

int load_driver() {
  std::call_once(g_driver_once, [] {
    auto get = [](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q;
      cudaError_t e = cudaGetDriverEntryPointByVersion(name, fn, 12000, cudaEnableDefault, &q);
      if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !*fn)
        g_driver_status = FMX_ERR_UNSUPPORTED;
    };
    get("cuStreamBatchMemOp", (void**)&g_batch);
    get("cuStreamGetCtx", (void**)&g_stream_ctx);
    get("cuCtxPushCurrent", (void**)&g_ctx_push);
    get("cuCtxPopCurrent", (void**)&g_ctx_pop);
    get("cuCtxGetCurrent", (void**)&g_ctx_current);
  });
  if (g_driver_status != FMX_OK)
    return fail(FMX_ERR_UNSUPPORTED, "driver entry points (stream mem ops / contexts) unavailable");
  return FMX_OK;
}

// Graph entry points (fmx_graph_*), loaded on first use.
typedef CUresult (*PFN_graphGetNodes)(CUgraph, CUgraphNode*, size_t*);
typedef CUresult (*PFN_nodeGetType)(CUgraphNode, CUgraphNodeType*);
typedef CUresult (*PFN_memopGet)(CUgraphNode, CUDA_BATCH_MEM_OP_NODE_PARAMS*);
typedef CUresult (*PFN_execMemopSet)(CUgraphExec, CUgraphNode, const CUDA_BATCH_MEM_OP_NODE_PARAMS*);
typedef CUresult (*PFN_addMemop)(CUgraphNode*, CUgraph, const CUgraphNode*, size_t,
                                 const CUDA_BATCH_MEM_OP_NODE_PARAMS*);
typedef CUresult (*PFN_nodeDeps)(CUgraphNode, CUgraphNode*, size_t*);
PFN_graphGetNodes g_graph_nodes = nullptr;
PFN_nodeGetType g_node_type = nullptr;
PFN_memopGet g_memop_get = nullptr;
PFN_execMemopSet g_exec_memop_set = nullptr;
PFN_addMemop g_add_memop = nullptr;
PFN_nodeDeps g_node_dependents = nullptr;
std::once_flag g_graph_once;
int g_graph_status = FMX_OK;

int load_graph_driver() {
  if (int rc = load_driver()) return rc;
  std::call_once(g_graph_once, [] {
    auto get = [](const char* name, void** fn) {
      cudaDriverEntryPointQueryResult q;
      cudaError_t e = cudaGetDriverEntryPointByVersion(name, fn, 12000, cudaEnableDefault, &q);
      if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !*fn)
        g_graph_status = FMX_ERR_UNSUPPORTED;
    };
    get("cuGraphGetNodes", (void**)&g_graph_nodes);
    get("cuGraphNodeGetType", (void**)&g_node_type);
    get("cuGraphBatchMemOpNodeGetParams", (void**)&g_memop_get);
    get("cuGraphExecBatchMemOpNodeSetParams", (void**)&g_exec_memop_set);
    get("cuGraphAddBatchMemOpNode", (void**)&g_add_memop);
    get("cuGraphNodeGetDependentNodes", (void**)&g_node_dependents);
  });
  if (g_graph_status != FMX_OK)
    return fail(FMX_ERR_UNSUPPORTED, "driver graph entry points (batch memop nodes) unavailable");
  return FMX_OK;
}

#define FMX_CUDA(call)                                                                    \
  do {                                                                                    \
    cudaError_t _e = (call);                                                              \
    if (_e != cudaSuccess)                                                                \
      return fail(FMX_ERR_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(_e), \
                  __FILE__, __LINE__);                                                    \
  } while (0)

// Default slice (bytes per (owner, contributor) slot) and pipeline depth.  With
// two ranks per communicator each round moves little, so rounds are longer and
// the ring deeper: 16 MiB x 4 slots (n=2: 6.36 -> 5.88 ms for 102 MB,
// profiles/r01/r3k); 4 MiB x 2 slots otherwise (n=7: 8 MiB and K=3 no better, r3g).
inline size_t default_slice_cap(int nranks) { return nranks <= 2 ? (16u << 20) : (4u << 20); }
inline int default_slots(int nranks) { return nranks <= 2 ? 4 : 2; }
// Default cap on data-slot bytes: the in-slots grow with n^2, so wide
// communicators get a larger budget (n = 56 on 8 GPUs: 326 KiB slices instead
// of 163 KiB, 6 rounds per ResNet-50 allreduce instead of 11).
inline size_t segment_budget(int nranks) { return nranks > 14 ? (2ull << 30) : (1ull << 30); }
constexpr int kBatchMax = 128;                  // memops per cuStreamBatchMemOp call

bool pid_alive(int pid) { return pid > 0 && (kill(pid, 0) == 0 || errno == EPERM); }

}  // namespace

namespace {

void unmap(fmx_comm* c) {
  if (c->base) munmap(c->base, c->total_bytes);
  c->base = nullptr;
  c->hdr = nullptr;
}

int grid_for(size_t work_items, int threads, int cap) {
  size_t g = (work_items + threads - 1) / threads;
  return (int)std::max<size_t>(1, std::min<size_t>(g, (size_t)cap));
}

enum StampKind { kStWaitPeers = 1, kStWaitRank, kStWaitEvent, kStCopy, kStReduce, kStSignal };

// Is a kernel profiler / checker injected into this process?  ncu (and the
// sanitizers) serialise kernel launches across processes behind one lock and
// drain the launching context first.  A collective's kernel queued behind a
// stream wait on a peer's flag then holds the lock while the peer - blocked
// on the same lock before the launch that would raise the flag - cannot
// proceed: a cross-process deadlock (the driver's ncu-instrumented smoke hung
// that way in round 1).  In serialize mode the host drains this rank's lanes
// before every kernel launch, so a launch never has pending dependencies; the
// schedule stays deadlock-free because its enqueue order is a valid
// single-FIFO schedule (tests/test_protocol_model.py).
bool profiler_injected() {
  if (const char* v = getenv("FMX_SERIALIZE")) return atoi(v) != 0;
  static const char* kVars[] = {"CUDA_INJECTION64_PATH", "NV_NSIGHT_INJECTION_TRANSPORT_TYPE",
                                "NSYS_PROFILING_SESSION_ID"};
  for (const char* k : kVars)
    if (getenv(k) && *getenv(k)) return true;
  return false;
}

class CudaSink final : public Sink {
 public:
  CudaSink(fmx_comm* c) : c_(c) {}

  // serialize mode: wait (on the host) for everything this rank enqueued so far
  // (not while capturing: nothing runs during a capture)
  int drain() {
    if (!c_->serialize || c_->cap_active) return FMX_OK;
    const cudaStream_t ss[4] = {c_->user, lane_stream(c_, 0), lane_stream(c_, 1),
                                lane_stream(c_, 2)};
    for (int i = 0; i < 4; ++i) FMX_CUDA(cudaStreamSynchronize(ss[i]));
    return FMX_OK;
  }

  // timeline probe: stamp the completion of the op just enqueued on `lane`
  int stamp(int lane, int kind, uint32_t info) {
    // (in a capture the stamp slots are baked: each replay rewrites them)
    if (!c_->stamps || c_->stamp_used >= c_->stamp_cap) return FMX_OK;
    if (int rc = drain()) return rc;
    fmx_stamp_kernel<<<1, 1, 0, lane_stream(c_, lane)>>>(c_->stamps + c_->stamp_used++,
                                                          (uint32_t)(lane << 8 | kind), info);
    FMX_CUDA(cudaGetLastError());
    return FMX_OK;
  }

  int copy_impl(int lane, const std::vector<PlanSeg>& segs, bool src_sys, bool use_kernel) {
    if (segs.empty()) return FMX_OK;
    cudaStream_t s = lane_stream(c_, lane);
    if (!use_kernel) {
      // copy engine; coalesce equal-size, equal-stride runs into one 2D copy
      size_t i = 0;
      while (i < segs.size()) {
        size_t k = 1;
        if (c_->copy2d && i + 1 < segs.size()) {
          const ptrdiff_t ds = segs[i + 1].dst - segs[i].dst, ss = segs[i + 1].src - segs[i].src;
          if (ds >= (ptrdiff_t)segs[i].bytes && ss >= (ptrdiff_t)segs[i].bytes && ds < (1ll << 31) &&
              ss < (1ll << 31))
            while (i + k < segs.size() && segs[i + k].bytes == segs[i].bytes &&
                   segs[i + k].dst - segs[i + k - 1].dst == ds &&
                   segs[i + k].src - segs[i + k - 1].src == ss)
              ++k;
          if (k > 1) {
            FMX_CUDA(cudaMemcpy2DAsync(segs[i].dst, (size_t)ds, segs[i].src, (size_t)ss,
                                       segs[i].bytes, k, cudaMemcpyDefault, s));
            i += k;
            continue;
          }
        }
        FMX_CUDA(cudaMemcpyAsync(segs[i].dst, segs[i].src, segs[i].bytes, cudaMemcpyDefault, s));
        ++i;
      }
      return FMX_OK;
    }
    return launch_copy(lane, segs, src_sys, nullptr, 0, nullptr);
  }

  // zero-copy copy kernel(s); with `flag` (a single launch) the kernel releases it,
  // electing the last CTA through the device counter `done`
  int launch_copy(int lane, const std::vector<PlanSeg>& segs, bool src_sys, uint32_t* flag,
                  uint32_t v, unsigned int* done) {
    cudaStream_t s = lane_stream(c_, lane);
    for (size_t i0 = 0; i0 < segs.size(); i0 += kMaxSegs) {
      if (int rc = drain()) return rc;
      CopyArgs a;
      memset(&a, 0, sizeof a);
      a.nseg = (int)std::min<size_t>(kMaxSegs, segs.size() - i0);
      a.src_sys = src_sys ? 1 : 0;
      a.flag = flag;
      a.flag_value = v;
      a.ctas_done = done;
      size_t maxb = 0;
      for (int k = 0; k < a.nseg; ++k) {
        a.seg[k] = CopySeg{segs[i0 + k].src, segs[i0 + k].dst, segs[i0 + k].bytes};
        maxb = std::max(maxb, a.seg[k].bytes);
      }
      constexpr int kThreads = 512, kU = 4;
      int gx = grid_for((maxb / 16 + kU - 1) / kU, kThreads, std::max(1, c_->copy_ctas / a.nseg));
      dim3 grid(gx, a.nseg);
      fmx_copy_kernel<kU><<<grid, kThreads, 0, s>>>(a);
      FMX_CUDA(cudaGetLastError());
      c_->launches++;
    }
    return FMX_OK;
  }

  int reduce_impl(int lane, const PlanReduce& r) {
    const ReduceArgs& a = r.args;
    if (a.len == 0) return FMX_OK;
    if (int rc = drain()) return rc;
    cudaStream_t s = lane_stream(c_, lane);
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    if (c_->timing && !c_->cap_active) {
      if (c_->timed_used == c_->timed.size()) {
        cudaEvent_t x, y;
        FMX_CUDA(cudaEventCreate(&x));
        FMX_CUDA(cudaEventCreate(&y));
        c_->timed.push_back({x, y});
      }
      t0 = c_->timed[c_->timed_used].first;
      t1 = c_->timed[c_->timed_used].second;
      c_->timed_used++;
      FMX_CUDA(cudaEventRecord(t0, s));
    }
    launch_reduce(a, r.dtype, r.aligned, s, c_->reduce_ctas);
    FMX_CUDA(cudaGetLastError());
    if (t1) FMX_CUDA(cudaEventRecord(t1, s));
    c_->launches++;
    return FMX_OK;
  }

  int signal_impl(int lane, int flag, uint32_t v) {
    CUstreamBatchMemOpParams op;
    memset(&op, 0, sizeof op);
    op.writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_32;
    op.writeValue.address = c_->flag_dev(c_->rank, flag);
    op.writeValue.value = v;
    op.writeValue.flags = CU_STREAM_WRITE_VALUE_DEFAULT;  // fence before the write
    return batch(lane, &op, 1);
  }

  int signal2_impl(int lane, int f0, uint32_t v0, int f1, uint32_t v1) {
    CUstreamBatchMemOpParams op[2];
    memset(op, 0, sizeof op);
    op[0].writeValue.operation = op[1].writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_32;
    op[0].writeValue.address = c_->flag_dev(c_->rank, f0);
    op[0].writeValue.value = v0;
    op[1].writeValue.address = c_->flag_dev(c_->rank, f1);
    op[1].writeValue.value = v1;
    return batch(lane, op, 2);
  }

  int wait_peers_impl(int lane, int flag, uint32_t v, int skip) {
    ops_.clear();
    for (int q = 0; q < c_->nranks; ++q)
      if (q != skip) ops_.push_back(wait_op(q, flag, v));
    for (size_t i = 0; i < ops_.size(); i += kBatchMax) {
      int rc = batch(lane, ops_.data() + i, (unsigned)std::min<size_t>(kBatchMax, ops_.size() - i));
      if (rc) return rc;
    }
    return FMX_OK;
  }

  int wait_rank_impl(int lane, int q, int flag, uint32_t v) {
    CUstreamBatchMemOpParams op = wait_op(q, flag, v);
    return batch(lane, &op, 1);
  }

  int d2d(int lane, void* dst, const void* src, size_t bytes, Annot, Annot) override {
    FMX_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, lane_stream(c_, lane)));
    return FMX_OK;
  }

  int record(int lane, int ev) override {
    FMX_CUDA(cudaEventRecord(c_->ev[ev], lane_stream(c_, lane)));
    c_->ev_cap[ev] = c_->cap_active;
    return FMX_OK;
  }

  // A wait on an event last recorded in another capture or on the eager
  // timeline is dropped (it cannot be captured, and is covered by the stream
  // order of graph launches plus the fence every replay ends with).
  int wait_event_impl(int lane, int ev) {
    if (c_->ev_cap[ev] != c_->cap_active) return FMX_OK;
    FMX_CUDA(cudaStreamWaitEvent(lane_stream(c_, lane), c_->ev[ev], 0));
    return FMX_OK;
  }

  // every op, then (timeline probe on) a stamp of its completion on its lane
  int copy(int lane, const std::vector<PlanSeg>& segs, bool src_sys, bool use_kernel) override {
    size_t bytes = 0;
    for (const PlanSeg& g : segs) bytes += g.bytes;
    int rc = copy_impl(lane, segs, src_sys, use_kernel);
    if (rc || segs.empty()) return rc;
    // Copy fence: a one-warp no-op kernel right after every copy-engine batch.
    // A stream memory op (flag signal / wait) directly behind a copy-engine
    // transfer takes a slow path on this B200 + MPS setup (13 back-to-back
    // 8 MiB allreduces on one stream: 162 ms; with the fence 32 ms), and the
    // fence also speeds up the plain allreduce (30.3 -> 28.1 ms) and the host
    // path (17.7 -> 16.6 ms) (profiles/r01/r2z_r3a).  FMX_COPY_FENCE=0: off.
    if (!use_kernel && c_->copy_fence) {
      if ((rc = drain())) return rc;
      fmx_nop_kernel<<<1, 32, 0, lane_stream(c_, lane)>>>();
      FMX_CUDA(cudaGetLastError());
      c_->launches++;
    }
    return stamp(lane, kStCopy, (uint32_t)std::min<size_t>(bytes, ~0u));
  }
  int copy_signal(int lane, const std::vector<PlanSeg>& segs, bool src_sys, bool use_kernel,
                  int flag, uint32_t v) override {
    // zero-copy copy kernel that releases the flag itself (one launch, no memop)
    // (not in a captured graph: every flag value must sit in a memop node that
    // fmx_graph_launch_prepare can re-base)
    if (!use_kernel || !c_->fuse_signal || !c_->ctas_done || segs.empty() ||
        segs.size() > (size_t)kMaxSegs || c_->stamps || c_->cap_active)
      return Sink::copy_signal(lane, segs, src_sys, use_kernel, flag, v);
    const uint32_t* fl = (const uint32_t*)c_->flag_dev(c_->rank, flag);
    // one counter per lane that fuses signals (stage copies on lane 0, the
    // one-shot publish on lane 1), so two fused copies never share a counter
    return launch_copy(lane, segs, src_sys, (uint32_t*)fl, v, c_->ctas_done + (lane == kLaneMain));
  }

  // the one-shot's OS_READY wait fused into its reduction (MPS ranks, messages up
  // to 16 KiB: 1 KiB at 7 ranks 0.049 -> 0.028 ms; at 64 KiB the spinning
  // CTAs cost more than the memop wait saves, 0.119 vs 0.096 ms, r02/r2h)
  int wait_reduce(int lane, const PlanReduce& r, int flag, uint32_t v, int skip) override {
    const size_t bytes = r.args.len * (r.dtype == FMX_FLOAT32 ? 4 : 2);
    if (!c_->spin_wait || c_->stamps || c_->cap_active || r.args.len == 0 || bytes > (16u << 10))
      return Sink::wait_reduce(lane, r, flag, v, skip);
    PlanReduce f = r;
    f.args.wait_flags = (const char*)c_->flag_dev(0, flag);
    f.args.wait_stride = (size_t)kFlagsPerRank * 64;
    f.args.wait_value = v;
    f.args.wait_skip = skip;
    return reduce(lane, f);
  }

  int reduce(int lane, const PlanReduce& r) override {
    int rc = reduce_impl(lane, r);
    return rc || r.args.len == 0 ? rc : stamp(lane, kStReduce, (uint32_t)r.args.len);
  }
  int signal(int lane, int flag, uint32_t v) override {
    int rc = signal_impl(lane, flag, v);
    return rc ? rc : stamp(lane, kStSignal, v);
  }
  int signal2(int lane, int f0, uint32_t v0, int f1, uint32_t v1) override {
    int rc = signal2_impl(lane, f0, v0, f1, v1);
    return rc ? rc : stamp(lane, kStSignal, v0);
  }
  int wait_peers(int lane, int flag, uint32_t v, int skip) override {
    int rc = wait_peers_impl(lane, flag, v, skip);
    return rc ? rc : stamp(lane, kStWaitPeers, v);
  }
  int wait_rank(int lane, int q, int flag, uint32_t v) override {
    int rc = wait_rank_impl(lane, q, flag, v);
    return rc ? rc : stamp(lane, kStWaitRank, v);
  }
  int wait_event(int lane, int ev) override {
    int rc = wait_event_impl(lane, ev);
    return rc ? rc : stamp(lane, kStWaitEvent, (uint32_t)ev);
  }

 private:
  CUstreamBatchMemOpParams wait_op(int q, int flag, uint32_t v) {
    CUstreamBatchMemOpParams op;
    memset(&op, 0, sizeof op);
    op.waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_32;
    op.waitValue.address = c_->flag_dev(q, flag);
    op.waitValue.value = v;
    op.waitValue.flags = CU_STREAM_WAIT_VALUE_GEQ;  // cyclic >=
    return op;
  }
  int batch(int lane, CUstreamBatchMemOpParams* ops, unsigned n) {
    CUresult r = g_batch((CUstream)lane_stream(c_, lane), n, ops, 0);
    if (r != CUDA_SUCCESS) return fail(FMX_ERR_CUDA, "cuStreamBatchMemOp failed (%d)", (int)r);
    return FMX_OK;
  }
  fmx_comm* c_;
  std::vector<CUstreamBatchMemOpParams> ops_;
};

// Lane objects (lane-0/2 streams, the lane events, the fork/join/done events,
// the timing pairs) live in the context of the caller's stream - a green
// context, an MPS client's, or the primary one - so every lane object lives
// where the caller's work lives.  On a change of context the old objects are
// destroyed in their own context after a host wait for the last collective
// (its `done`), so ordering carries over: the new context's events start
// unrecorded, and every wait on them is then rightly a no-op.
int release_lane_objects(fmx_comm* c) {
  if (!c->lane_ctx) return FMX_OK;
  if (g_ctx_push(c->lane_ctx) != CUDA_SUCCESS) return fail(FMX_ERR_CUDA, "cuCtxPushCurrent failed");
  int rc = FMX_OK;
  if (c->has_done && c->done_cap == 0 && cudaEventSynchronize(c->done) != cudaSuccess)
    rc = fail(FMX_ERR_CUDA, "pending collective failed: %s", cudaGetErrorString(cudaGetLastError()));
  if (c->graph_stream && cudaStreamSynchronize(c->graph_stream) != cudaSuccess && rc == FMX_OK)
    rc = fail(FMX_ERR_CUDA, "pending graph replay failed: %s", cudaGetErrorString(cudaGetLastError()));
  if (c->done) cudaEventDestroy(c->done);
  if (c->fork) cudaEventDestroy(c->fork);
  if (c->graph_ev) cudaEventDestroy(c->graph_ev);
  c->done = c->fork = c->graph_ev = nullptr;
  c->graph_stream = nullptr;
  for (int i = 0; i < kNumEvents; ++i) {
    if (c->ev[i]) cudaEventDestroy(c->ev[i]);
    c->ev[i] = nullptr;
  }
  for (auto& pr : c->timed) {
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
  c->timed.clear();
  c->timed_used = 0;
  for (int l = 0; l < 3; ++l) {
    if (l != 1 && c->lane[l]) cudaStreamDestroy(c->lane[l]);
    if (c->joined[l]) cudaEventDestroy(c->joined[l]);
    c->lane[l] = nullptr;
    c->joined[l] = nullptr;
  }
  CUcontext dummy;
  g_ctx_pop(&dummy);
  c->has_done = false;
  c->last_class = -1;
  c->last_main = nullptr;
  c->completion = nullptr;
  c->lane_ctx = nullptr;
  return rc;
}

// (Re)create the lane objects in `ctx` (pushed by the caller).
int make_lane_objects(fmx_comm* c, CUcontext ctx) {
  // lane priority (FMX_LANE_PRIORITY=1: highest) stays default: high-priority
  // lanes made the device-buffer allreduce 1.4x slower on the B200 under MPS
  // (profiles/r01/r2o) and did not help DP training (r2k)
  int lo_prio = 0, hi_prio = 0, prio = 0;
  FMX_CUDA(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
  if (const char* v = getenv("FMX_LANE_PRIORITY")) prio = atoi(v) ? hi_prio : 0;
  for (int l = 0; l < 3; ++l) {
    // extra lane streams only where the schedule uses them (FMX_LANES=1: none)
    const bool used = (l == 0 && c->nlanes >= 2) || (l == 2 && c->nlanes == 3);
    if (used) FMX_CUDA(cudaStreamCreateWithPriority(&c->lane[l], cudaStreamNonBlocking, prio));
    FMX_CUDA(cudaEventCreateWithFlags(&c->joined[l], cudaEventDisableTiming));
  }
  FMX_CUDA(cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming));
  FMX_CUDA(cudaEventCreateWithFlags(&c->done, cudaEventDisableTiming));
  FMX_CUDA(cudaEventCreateWithFlags(&c->graph_ev, cudaEventDisableTiming));
  for (int i = 0; i < kNumEvents; ++i) FMX_CUDA(cudaEventCreateWithFlags(&c->ev[i], cudaEventDisableTiming));
  c->lane_ctx = ctx;
  return FMX_OK;
}

// Run one collective: lane 1 runs on the main stream (the join stream if one
// is set, else the caller's), lanes 0 and 2 on two extra streams; all fork
// from the caller's stream (the input is ready there) and join into the main
// stream.  With a join stream (fmx_comm_set_join_stream) the caller's stream
// runs on while the collective completes, and the next device-buffer call's
// stage can overlap this call's gather (slot reuse across calls is covered by
// the plan's W / G events, which count rounds globally).  A host-path or broadcast call, or the first device call
// after one, waits for the previous collective to complete.  Every runtime
// call happens with the caller's stream context current (DDP calls hooks from
// autograd threads whose current context may be another one).
//   cls: 0 device-buffer allreduce / reduce-scatter / all-gather, 1 other,
//        2 device-buffer collective on lane 1 alone (the one-shot allreduce: no
//        extra streams forked or joined).
template <typename F>
int on_lanes(fmx_comm* c, cudaStream_t user, int cls, F&& body) {
  CUcontext ctx = nullptr;
  if (g_stream_ctx((CUstream)user, &ctx) != CUDA_SUCCESS || !ctx)
    return fail(FMX_ERR_CUDA, "cannot resolve the context of the caller's stream");
  if (g_ctx_push(ctx) != CUDA_SUCCESS) return fail(FMX_ERR_CUDA, "cuCtxPushCurrent failed");
  struct Pop {
    ~Pop() {
      CUcontext dummy;
      g_ctx_pop(&dummy);
    }
  } pop;
  int rc;
  // capture discipline: a captured collective must be announced
  // (fmx_graph_capture_begin) so its flag values can be re-based per replay
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  FMX_CUDA(cudaStreamIsCapturing(user, &cs));
  if (cs == cudaStreamCaptureStatusActive && !c->cap_active)
    return fail(FMX_ERR_INVALID_ARG, "collective on a capturing stream: call fmx_graph_capture_begin first");
  if (cs != cudaStreamCaptureStatusActive && c->cap_active)
    return fail(FMX_ERR_INVALID_ARG, "capture mode is on but the stream is not capturing");
  if (ctx != c->lane_ctx) {
    if (c->cap_active) return fail(FMX_ERR_INVALID_ARG, "context change inside a capture");
    if ((rc = release_lane_objects(c)) || (rc = make_lane_objects(c, ctx))) return rc;
  }
  // the first eager call after a graph replay on another stream is ordered after it
  if (!c->cap_active && c->graph_stream) {
    if (c->graph_stream != user) {
      FMX_CUDA(cudaEventRecord(c->graph_ev, c->graph_stream));
      FMX_CUDA(cudaStreamWaitEvent(user, c->graph_ev, 0));
    }
    c->graph_stream = nullptr;
  }
  c->user = user;
  cudaStream_t main = c->join_stream ? c->join_stream : user;  // lane 1 and the join target
  // extra lane streams in use: lane 0, and lane 2 with three lanes
  const bool single = cls == 2;
  if (single) cls = 0;
  std::vector<cudaStream_t> extra;
  // (join-stream mode: FMX_JOIN_LANES=2/3 keep the stage / gather lanes as
  // extra streams too - in a captured graph, parallel branches)
  const int jl = c->join_stream ? std::min(c->join_lanes, c->nlanes) : c->nlanes;
  if (jl >= 2 && c->nlanes >= 2 && !single) extra.push_back(c->lane[0]);
  if (jl == 3 && c->nlanes == 3 && !single) extra.push_back(c->lane[2]);
  // host-path / broadcast calls (and the first device call after one) wait for
  // the previous collective, whichever stream it joined (redundant, and free,
  // when it joined the caller's stream)
  // A change of main stream is a barrier too: lane 1 (HBM scratch slots) is
  // ordered across calls only while it stays on one stream.
  const bool barrier = c->has_done && c->done_cap == c->cap_active &&
                       (cls != 0 || c->last_class != 0 || main != c->last_main);
  std::vector<cudaStream_t> lanes_ = extra;
  if (main != user) lanes_.push_back(main);
  if (!lanes_.empty()) FMX_CUDA(cudaEventRecord(c->fork, user));
  for (cudaStream_t s : lanes_) FMX_CUDA(cudaStreamWaitEvent(s, c->fork, 0));
  if (barrier) {
    for (cudaStream_t s : extra) FMX_CUDA(cudaStreamWaitEvent(s, c->done, 0));
    FMX_CUDA(cudaStreamWaitEvent(main, c->done, 0));
  }
  rc = body();
  // completion: the lanes join the main stream (the caller's, or the join
  // stream, which then carries every lane); fmx_comm_completion_stream names it
  cudaStream_t target = main;
  c->completion = target;
  for (size_t l = 0; l < extra.size(); ++l) {
    FMX_CUDA(cudaEventRecord(c->joined[l], extra[l]));
    FMX_CUDA(cudaStreamWaitEvent(target, c->joined[l], 0));
  }
  if (rc) return rc;
  FMX_CUDA(cudaEventRecord(c->done, target));
  c->done_cap = c->cap_active;
  c->fenced = false;
  c->has_done = true;
  c->last_class = cls;
  c->last_main = main;
  return FMX_OK;
}

int check_comm(fmx_comm* c, bool needs_device = true) {
  if (!c || !c->hdr) return fail(FMX_ERR_INVALID_ARG, "invalid communicator");
  if (c->hdr->aborted.load(std::memory_order_acquire))
    return fail(FMX_ERR_ABORTED, "communicator was aborted");
  if (needs_device && c->transport == FMX_TRANSPORT_HOST)
    return fail(FMX_ERR_UNSUPPORTED, "host-only communicator has no device path");
  return FMX_OK;
}


}  // namespace

extern "C" {

int fmx_comm_init(fmx_comm_t* out, const char* job_key, int nranks, int rank,
                  const fmx_peer_info* self, int mig_aware, size_t slice_bytes, int nslots,
                  size_t host_bytes, int transport, double timeout_s) {
  if (!out || !job_key || !self) return fail(FMX_ERR_INVALID_ARG, "null argument");
  *out = nullptr;
  if (nranks < 1 || nranks > FMX_MAX_RANKS)
    return fail(FMX_ERR_INVALID_ARG, "nranks %d outside 1..%d", nranks, FMX_MAX_RANKS);
  if (rank < 0 || rank >= nranks || self->rank != rank)
    return fail(FMX_ERR_BAD_RANKS, "ranks must be 0..%d and distinct", nranks - 1);
  size_t klen = strlen(job_key);
  if (klen == 0 || klen > 100 || strchr(job_key, '/'))
    return fail(FMX_ERR_INVALID_ARG, "job_key must be 1..100 chars without '/'");
  if (nslots == 0) {
    nslots = default_slots(nranks);
    if (const char* v = getenv("FMX_SLOTS")) nslots = atoi(v);
  }
  if (nslots < 2 || nslots > FMX_MAX_SLOTS)
    return fail(FMX_ERR_INVALID_ARG, "nslots must be 2..%d", FMX_MAX_SLOTS);
  if (transport < FMX_TRANSPORT_AUTO || transport > FMX_TRANSPORT_HOST)
    return fail(FMX_ERR_INVALID_ARG, "bad transport %d", transport);
  if (timeout_s <= 0) timeout_s = 120.0;
  fmx_peer_info me = *self;
  int rc = fmx_check_peer(&me);
  if (rc) return rc;
  const bool host_only = transport == FMX_TRANSPORT_HOST;
  if (!host_only && (rc = load_driver())) return rc;

  auto* c = new fmx_comm();
  c->rank = rank;
  c->nranks = nranks;
  c->nslots = nslots;
  const std::string name = std::string("/fmx-") + job_key;
  const double t_end = now_s() + timeout_s;

  if (rank == 0) {
    size_t sb = slice_bytes;
    if (sb == 0) {
      size_t per = (size_t)c->nslots * ((size_t)nranks * nranks + 2 * nranks);
      sb = std::min(default_slice_cap(nranks), segment_budget(nranks) / per);
    }
    sb = std::max<size_t>(4096, sb / 4096 * 4096);
    const Proto proto = proto_from_env();
    Layout L = compute_layout(nranks, c->nslots, sb, host_bytes, (size_t)std::max(0, proto.oneshot_max));
    shm_unlink(name.c_str());  // stale segment of a crashed job with the same key
    int fd = shm_open(name.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
    if (fd < 0) {
      delete c;
      return fail(FMX_ERR_SHM, "shm_open(%s) failed: %s", name.c_str(), strerror(errno));
    }
    if (ftruncate(fd, (off_t)L.total) != 0) {
      close(fd);
      shm_unlink(name.c_str());
      delete c;
      return fail(FMX_ERR_SHM, "ftruncate(%zu) failed: %s", L.total, strerror(errno));
    }
    void* p = mmap(nullptr, L.total, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (p == MAP_FAILED) {
      shm_unlink(name.c_str());
      delete c;
      return fail(FMX_ERR_SHM, "mmap(%zu) failed: %s", L.total, strerror(errno));
    }
    c->base = (char*)p;
    c->total_bytes = L.total;
    Header* h = (Header*)p;
    h->version = kVersion;
    h->nranks = nranks;
    h->nslots = c->nslots;
    h->slice_bytes = sb;
    h->total_bytes = L.total;
    h->peers_off = L.peers_off;
    h->flags_off = L.flags_off;
    h->ar_in_off = L.ar_in_off;
    h->ar_out_off = L.ar_out_off;
    h->bc_off = L.bc_off;
    h->os_off = L.os_off;
    h->os_bytes = L.os_bytes;
    h->user_off = L.user_off;
    h->user_bytes = L.user_bytes;
    h->creator_pid = (int32_t)getpid();
    h->mig_aware = mig_aware ? 1 : 0;
    snprintf(h->job_key, sizeof h->job_key, "%s", job_key);
    h->proto = proto;  // every rank runs rank 0's schedule settings
    h->magic.store(kMagicReady, std::memory_order_release);
  } else {
    for (;;) {
      if (now_s() > t_end) {
        delete c;
        return fail(FMX_ERR_TIMEOUT, "timed out waiting for rank 0 to create %s", name.c_str());
      }
      int fd = shm_open(name.c_str(), O_RDWR, 0600);
      if (fd < 0) {
        usleep(1000);
        continue;
      }
      struct stat st;
      if (fstat(fd, &st) != 0 || (size_t)st.st_size < 4096) {
        close(fd);
        usleep(1000);
        continue;
      }
      void* p = mmap(nullptr, (size_t)st.st_size, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
      close(fd);
      if (p == MAP_FAILED) {
        usleep(1000);
        continue;
      }
      Header* h = (Header*)p;
      if (h->magic.load(std::memory_order_acquire) != kMagicReady || !pid_alive(h->creator_pid) ||
          h->total_bytes != (uint64_t)st.st_size || h->version != kVersion) {
        munmap(p, (size_t)st.st_size);
        usleep(1000);
        continue;
      }
      if (h->nranks != nranks) {
        const int theirs = h->nranks;  // read before the unmap
        munmap(p, (size_t)st.st_size);
        delete c;
        return fail(FMX_ERR_BAD_RANKS, "segment %s has %d ranks, caller says %d", name.c_str(),
                    theirs, nranks);
      }
      c->base = (char*)p;
      c->total_bytes = (size_t)st.st_size;
      break;
    }
  }
  Header* h = c->hdr = (Header*)c->base;
  c->slice_bytes = h->slice_bytes;
  c->nslots = h->nslots;  // rank 0's choice wins
  c->L = Layout{h->peers_off, h->flags_off, h->ar_in_off, h->ar_out_off, h->bc_off,
                h->os_off,    h->os_bytes,  h->user_off,   h->user_bytes, h->total_bytes};
  c->mig_aware = h->mig_aware;

  // publish this rank's PeerInfo
  PeerSlot* slots = (PeerSlot*)(c->base + c->L.peers_off);
  int expected = 0;
  slots[rank].info = me;
  slots[rank].pid = (int32_t)getpid();
  if (!slots[rank].state.compare_exchange_strong(expected, 1, std::memory_order_acq_rel)) {
    unmap(c);
    delete c;
    return fail(FMX_ERR_BAD_RANKS, "rank %d joined twice", rank);
  }
  h->arrived.fetch_add(1, std::memory_order_acq_rel);
  while (h->arrived.load(std::memory_order_acquire) < nranks) {
    if (h->aborted.load() || now_s() > t_end) {
      int code = h->aborted.load() ? FMX_ERR_ABORTED : FMX_ERR_TIMEOUT;
      int got = h->arrived.load();
      if (rank == 0) shm_unlink(name.c_str());
      unmap(c);
      delete c;
      return fail(code, "bootstrap: %d of %d ranks arrived", got, nranks);
    }
    usleep(200);
  }
  if (rank == 0) shm_unlink(name.c_str());  // everyone has it mapped: no stale name on crash

  c->peers.resize(nranks);
  for (int r = 0; r < nranks; ++r) c->peers[r] = slots[r].info;
  int a = -1, b = -1;
  rc = fmx_validate_peers(c->peers.data(), nranks, c->mig_aware, &a, &b);
  if (rc == FMX_OK) {
    std::vector<char> labels((size_t)nranks * FMX_BUS_ID_LEN);
    rc = fmx_topology(c->peers.data(), nranks, labels.data(), nullptr, nullptr, nullptr);
  }
  // One host only: peers on another host would need the NET transport
  // (select_transport, reference commsim.py:126-132); every rank sees the same
  // table, so every rank refuses the communicator the same way.
  for (int r = 1; rc == FMX_OK && r < nranks; ++r)
    if (c->peers[r].host_hash != c->peers[0].host_hash)
      rc = fail(FMX_ERR_UNSUPPORTED,
                "rank %d is on another host than rank 0 (host_hash differs): select_transport "
                "answers NET, and this library provides only the SHM transport of one host", r);
  if (rc != FMX_OK) {
    unmap(c);
    delete c;
    return rc;  // message / dup pair already set
  }

  c->transport = transport;  // AUTO stays AUTO: chosen per collective by size (use_zc)
  apply_proto(c, h->proto);  // rank 0's schedule settings (never per-rank env)
  if (host_only) {
    *out = c;
    return FMX_OK;
  }
  // NUMA placement by first touch, before anyone pins the segment (pinning
  // faults every page in on the pinning rank's node): each owner writes the
  // regions only it reads or writes - its in-slots [k][me][*], its out-slots
  // [k][me], its registered host buffer - so on a multi-socket host they land
  // on the node of the CPUs the launcher pinned the rank to (the GPU's node).
  {
    const size_t sb = c->slice_bytes, n = (size_t)nranks;
    for (int k = 0; k < c->nslots; ++k) {
      memset(c->base + c->in_off(k, rank, 0), 0, n * sb);
      memset(c->base + c->out_off(k, rank), 0, sb);
    }
    if (c->L.user_bytes) memset(c->base + c->user_region_off(rank), 0, c->L.user_bytes);
    h->touched.fetch_add(1, std::memory_order_acq_rel);
    while (h->touched.load(std::memory_order_acquire) < nranks) {
      if (h->aborted.load() || now_s() > t_end) {
        unmap(c);
        delete c;
        return fail(FMX_ERR_TIMEOUT, "bootstrap: a rank failed to initialise its regions");
      }
      usleep(200);
    }
  }
  // device mapping
  cudaError_t e = cudaHostRegister(c->base, c->total_bytes,
                                   cudaHostRegisterMapped | cudaHostRegisterPortable);
  if (e == cudaSuccess) {
    c->registered = true;
    e = cudaHostGetDevicePointer((void**)&c->dbase, c->base, 0);
  }
  // HBM scratch: CE contributions [n] (device path) / [2][n] fetch + [2][n] result replicas (host path)
  if (e == cudaSuccess) e = cudaMalloc((void**)&c->scratch, 4 * (size_t)nranks * c->slice_bytes);
  if (e == cudaSuccess) e = cudaMalloc((void**)&c->ctas_done, 2 * sizeof(unsigned int));
  if (e == cudaSuccess) e = cudaMemset(c->ctas_done, 0, 2 * sizeof(unsigned int));


  // local-only knobs (how this rank issues its copies; the protocol is unchanged)
  if (const char* v = getenv("FMX_COPY2D")) c->copy2d = atoi(v) != 0;
  if (const char* v = getenv("FMX_STAGE_AFTER_REDUCE")) c->stage_after_reduce = atoi(v) != 0;
  if (const char* v = getenv("FMX_STAGE_ZC")) c->stage_zc = atoi(v) != 0;
  // The next round's fetch on the gather lane pays off with few ranks per GPU,
  // where each round's reduction stores as much as the fetch moves (two ranks:
  // 1 GiB 53.6-54.5 vs 60.1-60.7 ms), not with seven (the extra stream per MPS
  // client costs more: 290 vs 281 ms, r02/r3r).  Ranks on my GPU = peers with
  // my bus id.
  {
    int same = 0;
    for (const fmx_peer_info& p : c->peers)
      if (strncmp(p.pcie_bus_id, c->peers[rank].pcie_bus_id, FMX_BUS_ID_LEN) == 0) ++same;
    c->fetch_lane = same <= 2;
  }
  if (const char* v = getenv("FMX_FETCH_LANE")) c->fetch_lane = atoi(v) != 0;
  if (const char* v = getenv("FMX_RCE_ROUNDS")) c->rce_rounds = std::max(1, atoi(v));
  if (const char* v = getenv("FMX_COPY_FENCE")) c->copy_fence = atoi(v) != 0;
  if (const char* v = getenv("FMX_JOIN_LANES")) c->join_lanes = std::max(1, std::min(3, atoi(v)));
  if (const char* v = getenv("FMX_FUSE_SIGNAL")) c->fuse_signal = atoi(v) != 0;
  if (const char* v = getenv("FMX_COPY_CTAS")) c->copy_ctas = std::max(1, std::min(atoi(v), 1184));
  if (const char* v = getenv("FMX_REDUCE_CTAS")) c->reduce_ctas = std::max(1, std::min(atoi(v), kReduceGridCap));
  c->serialize = profiler_injected();
  // The one-shot may fuse its flag wait into the reduction (spinning CTAs) only
  // where ranks run concurrently - MPS clients; never time-sliced contexts
  // (green / plain processes), and never under a kernel profiler, whose
  // serialised launches would deadlock on a spinning kernel.
  {
    int dev = 0, mps = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&mps, cudaDevAttrMpsEnabled, dev) == cudaSuccess)
      c->spin_wait = mps != 0 && !c->serialize;
    cudaGetLastError();
    if (const char* v = getenv("FMX_SPIN_WAIT")) c->spin_wait = atoi(v) != 0 && !c->serialize;
  }
  if (e != cudaSuccess) {
    h->aborted.store(1);
    fail(FMX_ERR_CUDA, "device mapping of %zu-byte segment failed: %s", c->total_bytes,
         cudaGetErrorString(e));
    if (c->registered) cudaHostUnregister(c->base);
    if (c->scratch) cudaFree(c->scratch);
    if (c->ctas_done) cudaFree(c->ctas_done);
    unmap(c);
    delete c;
    return FMX_ERR_CUDA;
  }
  h->mapped.fetch_add(1, std::memory_order_acq_rel);
  while (h->mapped.load(std::memory_order_acquire) < nranks) {
    if (h->aborted.load() || now_s() > t_end) {
      int code = h->aborted.load() ? FMX_ERR_ABORTED : FMX_ERR_TIMEOUT;
      fmx_comm_destroy(c);
      return fail(code, "bootstrap: a rank failed to map the segment");
    }
    usleep(200);
  }
  *out = c;
  return FMX_OK;
}

int fmx_allreduce(fmx_comm_t c, const void* send, void* recv, size_t count, int dtype, int op,
                  float factor, void* stream) {
  int rc = check_comm(c);
  if (rc) return rc;
  if (dtype != FMX_FLOAT32 && dtype != FMX_BFLOAT16)
    return fail(FMX_ERR_INVALID_ARG, "bad dtype %d", dtype);
  if (op < FMX_OP_SUM || op > FMX_OP_PREMUL_SUM) return fail(FMX_ERR_INVALID_ARG, "bad op %d", op);
  if (op != FMX_OP_SUM && !std::isfinite(factor))
    return fail(FMX_ERR_INVALID_ARG, "factor must be finite");
  if (count == 0) return FMX_OK;
  if (!send || !recv) return fail(FMX_ERR_INVALID_ARG, "null buffer");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t esz = dtype == FMX_FLOAT32 ? 4 : 2;
  const bool aligned = (((uintptr_t)send | (uintptr_t)recv) & 15) == 0;
  CudaSink sink(c);
  if (c->nranks == 1) {  // nothing to exchange: apply the scale convention locally
    return on_lanes(c, s, 0, [&]() -> int {
      if (op == FMX_OP_SUM) {
        if (send != recv)
          FMX_CUDA(cudaMemcpyAsync(recv, send, count * esz, cudaMemcpyDeviceToDevice, lane_stream(c, kLaneMain)));
        return FMX_OK;
      }
      PlanReduce pr;
      memset(&pr.args, 0, sizeof pr.args);
      pr.args.src[0] = (const char*)send;
      pr.args.nsrc = 1;
      pr.args.out_dev = (char*)recv;
      pr.args.len = count;
      pr.args.op = op;
      pr.args.factor = factor;
      pr.dtype = dtype;
      pr.aligned = aligned;
      return sink.reduce(kLaneMain, pr);
    });
  }
  // (a deferred gather still pending runs on the gather lane first: then the
  // one-shot forks and joins the extra lanes like any pipelined call)
  if (c->use_oneshot(count * esz))
    return on_lanes(c, s, c->pending ? 0 : 2, [&]() {
      return plan_allreduce_oneshot(c, sink, (const char*)send, (char*)recv, count, dtype, op,
                                    factor, aligned);
    });
  return on_lanes(c, s, 0, [&]() {
    return plan_allreduce(c, sink, (const char*)send, (char*)recv, count, dtype, op, factor,
                          aligned);
  });
}

int fmx_allreduce_shard(fmx_comm_t c, size_t count, int dtype, size_t* offset, size_t* len) {
  if (!c || !offset || !len) return fail(FMX_ERR_INVALID_ARG, "null argument");
  if (dtype != FMX_FLOAT32 && dtype != FMX_BFLOAT16)
    return fail(FMX_ERR_INVALID_ARG, "bad dtype %d", dtype);
  if (c->nranks == 1 || count == 0) {
    *offset = 0;
    *len = count;
    return FMX_OK;
  }
  const Geometry g = allreduce_geometry(c, count, dtype);
  const size_t lo = std::min(count, (size_t)c->rank * g.chunk);
  *offset = lo;
  *len = std::min(g.chunk, count - lo);
  return FMX_OK;
}

int fmx_allreduce_sgd(fmx_comm_t c, const void* grad, void* param, void* momentum, size_t count,
                      int op, float factor, const fmx_sgd* sgd, void* stream) {
  int rc = check_comm(c);
  if (rc) return rc;
  if (!sgd || !grad || !param) return fail(FMX_ERR_INVALID_ARG, "null argument");
  if (op != FMX_OP_SUM && op != FMX_OP_PREMUL_SUM)
    return fail(FMX_ERR_INVALID_ARG, "fused SGD takes op SUM or PREMUL_SUM");
  if (op != FMX_OP_SUM && !std::isfinite(factor)) return fail(FMX_ERR_INVALID_ARG, "factor must be finite");
  if (grad == param) return fail(FMX_ERR_INVALID_ARG, "gradient and parameter buffers must differ");
  if (sgd->momentum != 0.f && !momentum) return fail(FMX_ERR_INVALID_ARG, "momentum buffer required");
  if (count == 0) return FMX_OK;
  SgdEpi e{(char*)(sgd->momentum != 0.f ? momentum : nullptr), sgd->lr, sgd->momentum,
           sgd->dampening, sgd->weight_decay, sgd->nesterov, sgd->first_step};
  const bool aligned = (((uintptr_t)grad | (uintptr_t)param | (uintptr_t)e.mom) & 15) == 0;
  CudaSink sink(c);
  if (c->nranks == 1) {  // my shard is the whole buffer: the step alone
    return on_lanes(c, (cudaStream_t)stream, 0, [&]() -> int {
      PlanReduce pr;
      memset(&pr.args, 0, sizeof pr.args);
      pr.args.src[0] = (const char*)grad;
      pr.args.nsrc = 1;
      pr.args.out_dev = (char*)param;
      pr.args.len = count;
      pr.args.op = op;
      pr.args.factor = factor;
      pr.args.sgd = 1;
      pr.args.mom = e.mom;
      pr.args.lr = e.lr;
      pr.args.mu = e.mu;
      pr.args.damp = e.damp;
      pr.args.wd = e.wd;
      pr.args.nesterov = e.nesterov;
      pr.args.init = e.init;
      pr.dtype = FMX_FLOAT32;
      pr.aligned = aligned;
      return sink.reduce(kLaneMain, pr);
    });
  }
  c->sgd = &e;  // the pipelined schedule (never the one-shot: the step runs on owners)
  rc = on_lanes(c, (cudaStream_t)stream, 0, [&]() {
    return plan_allreduce(c, sink, (const char*)grad, (char*)param, count, FMX_FLOAT32, op,
                          factor, aligned);
  });
  c->sgd = nullptr;
  return rc;
}

// Shared argument checks of the dtype / op / factor triple.
static int check_reduction_args(int dtype, int op, float factor) {
  if (dtype != FMX_FLOAT32 && dtype != FMX_BFLOAT16)
    return fail(FMX_ERR_INVALID_ARG, "bad dtype %d", dtype);
  if (op < FMX_OP_SUM || op > FMX_OP_PREMUL_SUM) return fail(FMX_ERR_INVALID_ARG, "bad op %d", op);
  if (op != FMX_OP_SUM && !std::isfinite(factor))
    return fail(FMX_ERR_INVALID_ARG, "factor must be finite");
  return FMX_OK;
}

int fmx_reduce_scatter(fmx_comm_t c, const void* send, void* recv, size_t recvcount, int dtype,
                       int op, float factor, void* stream) {
  int rc = check_comm(c);
  if (rc || (rc = check_reduction_args(dtype, op, factor))) return rc;
  if (recvcount == 0) return FMX_OK;
  if (!send || !recv) return fail(FMX_ERR_INVALID_ARG, "null buffer");
  const size_t esz = dtype == FMX_FLOAT32 ? 4 : 2;
  const bool aligned = (((uintptr_t)send | (uintptr_t)recv) & 15) == 0 && (recvcount * esz) % 16 == 0;
  CudaSink sink(c);
  return on_lanes(c, (cudaStream_t)stream, 0, [&]() -> int {
    if (c->nranks == 1) {  // my chunk is the whole buffer: apply the scale convention
      PlanReduce pr;
      memset(&pr.args, 0, sizeof pr.args);
      pr.args.src[0] = (const char*)send;
      pr.args.nsrc = 1;
      pr.args.out_dev = (char*)recv;
      pr.args.len = recvcount;
      pr.args.op = op;
      pr.args.factor = factor;
      pr.dtype = dtype;
      pr.aligned = (((uintptr_t)send | (uintptr_t)recv) & 15) == 0;
      return sink.reduce(kLaneMain, pr);
    }
    return plan_allreduce(c, sink, (const char*)send, (char*)recv, recvcount, dtype, op, factor,
                          aligned, kReduceScatter);
  });
}

int fmx_allgather(fmx_comm_t c, const void* send, void* recv, size_t sendcount, int dtype,
                  void* stream) {
  int rc = check_comm(c);
  if (rc) return rc;
  if (dtype != FMX_FLOAT32 && dtype != FMX_BFLOAT16)
    return fail(FMX_ERR_INVALID_ARG, "bad dtype %d", dtype);
  if (sendcount == 0) return FMX_OK;
  if (!send || !recv) return fail(FMX_ERR_INVALID_ARG, "null buffer");
  const size_t esz = dtype == FMX_FLOAT32 ? 4 : 2;
  CudaSink sink(c);
  return on_lanes(c, (cudaStream_t)stream, 0, [&]() -> int {
    if (c->nranks == 1) {
      if (send != recv)
        FMX_CUDA(cudaMemcpyAsync(recv, send, sendcount * esz, cudaMemcpyDeviceToDevice,
                                 lane_stream(c, kLaneMain)));
      return FMX_OK;
    }
    return plan_allreduce(c, sink, (const char*)send, (char*)recv, sendcount, dtype, FMX_OP_SUM,
                          1.0f, true, kAllgather);
  });
}

int fmx_reduce_local(const void* const* srcs, int nsrc, uint64_t sys_mask, void* dst,
                     void* dst_sys, size_t count, int dtype, int op, float factor, void* stream) {
  if (!srcs || nsrc < 1 || nsrc > FMX_MAX_RANKS || !dst)
    return fail(FMX_ERR_INVALID_ARG, "bad arguments");
  if (dtype != FMX_FLOAT32 && dtype != FMX_BFLOAT16)
    return fail(FMX_ERR_INVALID_ARG, "bad dtype %d", dtype);
  if (op < FMX_OP_SUM || op > FMX_OP_PREMUL_SUM) return fail(FMX_ERR_INVALID_ARG, "bad op %d", op);
  if (count == 0) return FMX_OK;
  ReduceArgs a;
  memset(&a, 0, sizeof a);
  uintptr_t bits = (uintptr_t)dst | (uintptr_t)dst_sys;
  for (int q = 0; q < nsrc; ++q) {
    if (!srcs[q]) return fail(FMX_ERR_INVALID_ARG, "null source %d", q);
    a.src[q] = (const char*)srcs[q];
    bits |= (uintptr_t)srcs[q];
  }
  a.nsrc = nsrc;
  a.sys_mask = sys_mask;
  a.out_dev = (char*)dst;
  a.out_sys = (char*)dst_sys;
  a.len = count;
  a.op = op;
  a.factor = factor;
  launch_reduce(a, dtype, (bits & 15) == 0, (cudaStream_t)stream);
  FMX_CUDA(cudaGetLastError());
  return FMX_OK;
}

int fmx_host_buffer(fmx_comm_t c, int rank, void** ptr, size_t* bytes) {
  if (!c || !c->base || !ptr || rank < 0 || rank >= c->nranks)
    return fail(FMX_ERR_INVALID_ARG, "bad arguments");
  *ptr = c->base + c->user_region_off(rank);
  if (bytes) *bytes = c->L.user_bytes;
  return FMX_OK;
}

int fmx_allreduce_host(fmx_comm_t c, size_t offset, size_t count, int dtype, int op, float factor,
                       void* stream) {
  int rc = check_comm(c);
  if (rc) return rc;
  if (dtype != FMX_FLOAT32 && dtype != FMX_BFLOAT16)
    return fail(FMX_ERR_INVALID_ARG, "bad dtype %d", dtype);
  if (op < FMX_OP_SUM || op > FMX_OP_PREMUL_SUM) return fail(FMX_ERR_INVALID_ARG, "bad op %d", op);
  if (op != FMX_OP_SUM && !std::isfinite(factor))
    return fail(FMX_ERR_INVALID_ARG, "factor must be finite");
  const size_t esz = dtype == FMX_FLOAT32 ? 4 : 2;
  if (offset % 16 || offset + count * esz > c->L.user_bytes)
    return fail(FMX_ERR_INVALID_ARG, "host range [%zu, +%zu) outside the %zu-byte region (16-B aligned offset required)",
                offset, count * esz, (size_t)c->L.user_bytes);
  if (count == 0) return FMX_OK;
  CudaSink sink(c);
  return on_lanes(c, (cudaStream_t)stream, 1, [&]() {
    return plan_allreduce_host(c, sink, offset, count, dtype, op, factor);
  });
}

int fmx_broadcast(fmx_comm_t c, const void* send, void* recv, size_t count, int dtype, int root,
                  void* stream) {
  int rc = check_comm(c);
  if (rc) return rc;
  if (dtype != FMX_FLOAT32 && dtype != FMX_BFLOAT16)
    return fail(FMX_ERR_INVALID_ARG, "bad dtype %d", dtype);
  if (root < 0 || root >= c->nranks) return fail(FMX_ERR_INVALID_ARG, "bad root %d", root);
  if (count == 0) return FMX_OK;
  const size_t esz = dtype == FMX_FLOAT32 ? 4 : 2;
  if (!recv || (c->rank == root && !send)) return fail(FMX_ERR_INVALID_ARG, "null buffer");
  cudaStream_t s = (cudaStream_t)stream;
  CudaSink sink(c);
  if (c->nranks == 1) {
    return on_lanes(c, s, 1, [&]() -> int {
      if (send != recv)
        FMX_CUDA(cudaMemcpyAsync(recv, send, count * esz, cudaMemcpyDeviceToDevice, lane_stream(c, kLaneMain)));
      return FMX_OK;
    });
  }
  return on_lanes(c, s, 1, [&]() {
    return plan_broadcast(c, sink, (const char*)send, (char*)recv, count, dtype, root);
  });
}

int fmx_barrier(fmx_comm_t c, double timeout_s) {
  int rc = check_comm(c, false);
  if (rc) return rc;
  if (timeout_s <= 0) timeout_s = 120.0;
  const double t_end = now_s() + timeout_s;
  c->barrier_gen++;
  const int64_t target = c->barrier_gen * c->nranks;
  c->hdr->barrier_count.fetch_add(1, std::memory_order_acq_rel);
  while (c->hdr->barrier_count.load(std::memory_order_acquire) < target) {
    if (c->hdr->aborted.load()) return fail(FMX_ERR_ABORTED, "communicator was aborted");
    if (now_s() > t_end) return fail(FMX_ERR_TIMEOUT, "barrier timed out");
    std::this_thread::yield();
  }
  return FMX_OK;
}

int fmx_comm_destroy(fmx_comm_t c) {
  if (!c) return fail(FMX_ERR_INVALID_ARG, "invalid communicator");
  int rc = g_ctx_push ? release_lane_objects(c) : FMX_OK;
  drop_pending(c);
  if (c->scratch) cudaFree(c->scratch);
  if (c->stamps) cudaFree(c->stamps);
  if (c->ctas_done) cudaFree(c->ctas_done);
  if (c->registered) cudaHostUnregister(c->base);
  if (c->hdr) c->hdr->departed.fetch_add(1);
  unmap(c);
  delete c;
  return rc;
}

int fmx_comm_abort(fmx_comm_t c) {
  if (!c || !c->hdr) return fail(FMX_ERR_INVALID_ARG, "invalid communicator");
  c->hdr->aborted.store(1, std::memory_order_release);
  // Release every pending stream wait of every rank: raise all counters far
  // ahead (waits compare cyclic >=, so +2^29 satisfies any outstanding
  // target).  A GPU that still has a queued flag signal can write a smaller,
  // absolute value back after the raise and park a peer again, so the raise is
  // re-asserted until every flag stayed up for a quiet period (bounded), and
  // abort may be issued again at any time - e.g. after the local streams
  // drained: the raised targets are remembered, so repeating it is idempotent.
  const size_t nf = (size_t)c->nranks * kFlagsPerRank;
  if (c->abort_target.size() != nf) {
    c->abort_target.resize(nf);
    for (int r = 0; r < c->nranks; ++r)
      for (int f = 0; f < kFlagsPerRank; ++f)
        c->abort_target[(size_t)r * kFlagsPerRank + f] = *c->flag_host(r, f) + (1u << 29);
  }
  const double t_end = now_s() + 0.5;
  double quiet_since = now_s();
  while (now_s() < t_end && now_s() - quiet_since < 0.05) {
    for (int r = 0; r < c->nranks; ++r)
      for (int f = 0; f < kFlagsPerRank; ++f) {
        uint32_t* p = (uint32_t*)c->flag_host(r, f);
        const uint32_t want = c->abort_target[(size_t)r * kFlagsPerRank + f];
        const uint32_t v = __atomic_load_n(p, __ATOMIC_ACQUIRE);
        if ((int32_t)(v - want) < 0) {
          __atomic_store_n(p, want, __ATOMIC_RELEASE);
          quiet_since = now_s();
        }
      }
    std::this_thread::yield();
  }
  return FMX_OK;
}

int fmx_comm_rank(fmx_comm_t c, int* rank) {
  if (!c || !rank) return fail(FMX_ERR_INVALID_ARG, "null argument");
  *rank = c->rank;
  return FMX_OK;
}

int fmx_comm_count(fmx_comm_t c, int* nranks) {
  if (!c || !nranks) return fail(FMX_ERR_INVALID_ARG, "null argument");
  *nranks = c->nranks;
  return FMX_OK;
}

int fmx_comm_peer(fmx_comm_t c, int rank, fmx_peer_info* out) {
  if (!c || !out || rank < 0 || rank >= c->nranks) return fail(FMX_ERR_INVALID_ARG, "bad rank");
  *out = c->peers[rank];
  return FMX_OK;
}

int fmx_comm_config(fmx_comm_t c, size_t* slice_bytes, int* transport, size_t* shm_bytes) {
  if (!c) return fail(FMX_ERR_INVALID_ARG, "invalid communicator");
  if (slice_bytes) *slice_bytes = c->slice_bytes;
  if (transport) *transport = c->transport;
  if (shm_bytes) *shm_bytes = c->total_bytes;
  return FMX_OK;
}

int fmx_comm_flags(fmx_comm_t c, uint32_t* out, int cap) {
  if (!c || !c->base || !out || cap < c->nranks * 4)
    return fail(FMX_ERR_INVALID_ARG, "bad arguments");
  for (int r = 0; r < c->nranks; ++r)
    for (int f = 0; f < 4; ++f) out[r * 4 + f] = *c->flag_host(r, f);
  return FMX_OK;
}

int fmx_comm_monitor(fmx_comm_t c, double seconds, uint64_t* out, size_t cap, size_t* n_out) {
  if (!c || !c->base || !out || !n_out) return fail(FMX_ERR_INVALID_ARG, "bad arguments");
  const int n = c->nranks, nf = kStagedTo + n;
  std::vector<uint32_t> last((size_t)n * nf);
  for (int r = 0; r < n; ++r)
    for (int f = 0; f < nf; ++f) last[(size_t)r * nf + f] = *c->flag_host(r, f);
  size_t k = 0;
  const double t0 = now_s(), t_end = t0 + seconds;
  double t = t0;
  while (t < t_end && k + 2 <= cap) {
    for (int r = 0; r < n; ++r)
      for (int f = 0; f < nf; ++f) {
        const uint32_t v = *c->flag_host(r, f);
        uint32_t& l = last[(size_t)r * nf + f];
        if (v != l && k + 2 <= cap) {
          l = v;
          out[k++] = (uint64_t)((t - t0) * 1e9);
          out[k++] = ((uint64_t)r << 48) | ((uint64_t)f << 32) | v;
        }
      }
    t = now_s();
  }
  *n_out = k / 2;
  return FMX_OK;
}

int fmx_comm_set_join_stream(fmx_comm_t c, void* stream) {
  if (!c) return fail(FMX_ERR_INVALID_ARG, "invalid communicator");
  c->join_stream = (cudaStream_t)stream;
  return FMX_OK;
}

int fmx_comm_completion_stream(fmx_comm_t c, void** stream) {
  if (!c || !stream) return fail(FMX_ERR_INVALID_ARG, "null argument");
  *stream = (void*)c->completion;
  return FMX_OK;
}

int fmx_comm_set_timing(fmx_comm_t c, int on) {
  if (!c) return fail(FMX_ERR_INVALID_ARG, "invalid communicator");
  c->timing = on != 0;
  c->timed_used = 0;
  return FMX_OK;
}

int fmx_comm_kernel_time(fmx_comm_t c, double* total_ms, uint64_t* count) {
  if (!c || !total_ms || !count) return fail(FMX_ERR_INVALID_ARG, "null argument");
  double sum = 0;
  const bool pushed = c->lane_ctx && g_ctx_push(c->lane_ctx) == CUDA_SUCCESS;
  struct Pop {
    bool on;
    ~Pop() {
      CUcontext d;
      if (on) g_ctx_pop(&d);
    }
  } pop{pushed};
  for (size_t i = 0; i < c->timed_used; ++i) {
    FMX_CUDA(cudaEventSynchronize(c->timed[i].second));
    float ms = 0;
    FMX_CUDA(cudaEventElapsedTime(&ms, c->timed[i].first, c->timed[i].second));
    sum += ms;
  }
  *total_ms = sum;
  *count = c->timed_used;
  return FMX_OK;
}

int fmx_comm_set_stamps(fmx_comm_t c, size_t capacity) {
  if (!c) return fail(FMX_ERR_INVALID_ARG, "invalid communicator");
  const bool pushed = c->lane_ctx && g_ctx_push(c->lane_ctx) == CUDA_SUCCESS;
  struct Pop {
    bool on;
    ~Pop() {
      CUcontext d;
      if (on) g_ctx_pop(&d);
    }
  } pop{pushed};
  if (c->stamps) {
    FMX_CUDA(cudaDeviceSynchronize());
    FMX_CUDA(cudaFree(c->stamps));
  }
  c->stamps = nullptr;
  c->stamp_cap = c->stamp_used = 0;
  if (capacity) {
    FMX_CUDA(cudaMalloc((void**)&c->stamps, capacity * sizeof(Stamp)));
    c->stamp_cap = capacity;
  }
  return FMX_OK;
}

int fmx_comm_stamp(fmx_comm_t c, void* stream, uint32_t info) {
  if (!c) return fail(FMX_ERR_INVALID_ARG, "invalid communicator");
  if (!c->stamps || c->stamp_used >= c->stamp_cap) return FMX_OK;
  fmx_stamp_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(c->stamps + c->stamp_used++,
                                                       (uint32_t)(15u << 8 | 7u), info);
  FMX_CUDA(cudaGetLastError());
  return FMX_OK;
}

int fmx_comm_stamps(fmx_comm_t c, uint64_t* out, size_t cap, size_t* n_out) {
  if (!c || !out || !n_out) return fail(FMX_ERR_INVALID_ARG, "null argument");
  const size_t n = std::min(c->stamp_used, cap / 2);
  *n_out = n;
  if (!n) return FMX_OK;
  const bool pushed = c->lane_ctx && g_ctx_push(c->lane_ctx) == CUDA_SUCCESS;
  struct Pop {
    bool on;
    ~Pop() {
      CUcontext d;
      if (on) g_ctx_pop(&d);
    }
  } pop{pushed};
  std::vector<Stamp> h(n);
  FMX_CUDA(cudaDeviceSynchronize());
  FMX_CUDA(cudaMemcpy(h.data(), c->stamps, n * sizeof(Stamp), cudaMemcpyDeviceToHost));
  for (size_t i = 0; i < n; ++i) {
    out[2 * i] = h[i].t_ns;
    out[2 * i + 1] = ((uint64_t)h[i].tag << 32) | h[i].info;
  }
  return FMX_OK;
}

// ---- CUDA graphs ---------------------------------------------------------------
//
// A training step that contains collectives can be captured into one CUDA
// graph and replayed (ddp.ShmDataParallel).  Eager launches make the GPU read
// every launch's work from host memory, and those reads queue behind the
// exchange's own host-link traffic: ResNet-50 fwd+bwd 10.7 -> 18.2 ms under
// D2H copy traffic eager, 8.5 -> 8.7 ms as a graph (profiles/r02/r2o).
//
// Graph nodes bake their parameters, and a collective's flag values are round
// counters.  So: capture_begin snapshots the counters; every captured signal /
// wait is a batch-memop node; capture_end appends a fence (signal FENCE, wait
// for every peer's FENCE) after every leaf, finds the memop nodes on this
// communicator's flags and rolls the counters back (nothing ran);
// launch_prepare re-bases each node's values by how far its counter moved since
// the capture and advances the counters by one replay.  Slot addresses stay as
// captured: every replay starts with no peer touching any slot (the previous
// replay's fence; an eager fence first if collectives ran since), so the
// schedule inside a replay is the model-checked one, shifted in round numbers
// only.  Replays (and eager calls after them) are ordered by stream order.

namespace {

int flag_counter(const fmx_comm* c, CUdeviceptr addr) {
  const CUdeviceptr base = c->flag_dev(0, 0);
  const CUdeviceptr end = base + (CUdeviceptr)c->nranks * kFlagsPerRank * 64;
  if (addr < base || addr >= end) return -1;
  const int f = (int)(((addr - base) / 64) % kFlagsPerRank);
  if (f == kStaged || f == kReduced || f >= kStagedTo) return kCtrAr;
  if (f == kOsReady) return kCtrOs;
  if (f == kBcStaged || f == kBcDone) return kCtrBc;
  if (f == kFence) return kCtrFence;
  return -2;
}

struct CtxPush {
  bool on = false;
  explicit CtxPush(CUcontext ctx) { on = ctx && g_ctx_push && g_ctx_push(ctx) == CUDA_SUCCESS; }
  ~CtxPush() {
    CUcontext d;
    if (on) g_ctx_pop(&d);
  }
};

}  // namespace

int fmx_comm_fence(fmx_comm_t c, void* stream) {
  int rc = check_comm(c);
  if (rc) return rc;
  CudaSink sink(c);
  rc = on_lanes(c, (cudaStream_t)stream, 1, [&]() -> int {
    return c->nranks == 1 ? FMX_OK : plan_fence(c, sink);
  });
  if (rc) return rc;
  if (!c->cap_active) c->fenced = true;
  return FMX_OK;
}

int fmx_comm_set_defer(fmx_comm_t c, int on) {
  if (!c) return fail(FMX_ERR_INVALID_ARG, "invalid communicator");
  if (!on && c->pending) return fail(FMX_ERR_INVALID_ARG, "flush the deferred gather first");
  c->defer_gather = on != 0;
  return FMX_OK;
}

int fmx_comm_flush(fmx_comm_t c, void* stream) {
  int rc = check_comm(c);
  if (rc || !c->pending) return rc;
  CudaSink sink(c);
  return on_lanes(c, (cudaStream_t)stream, 0, [&]() { return plan_flush(c, sink); });
}

int fmx_graph_capture_begin(fmx_comm_t c) {
  int rc = check_comm(c);
  if (rc) return rc;
  if (c->cap_active) return fail(FMX_ERR_INVALID_ARG, "a capture is already active");
  if (c->pending) return fail(FMX_ERR_INVALID_ARG, "flush the deferred gather before a capture");
  if ((rc = load_graph_driver())) return rc;
  if (c->has_done && c->done_cap == 0 && c->lane_ctx) {
    // eager work still in flight: the captured collectives drop their waits
    // on eager events, and a replay is ordered after it by launch_prepare
    CtxPush push(c->lane_ctx);
    FMX_CUDA(cudaEventSynchronize(c->done));
  }
  if (!c->lane_ctx) {
    // no collective yet: the lane streams / events are created now, in the
    // current context (creating them inside the capture is not allowed); a
    // capture on a stream of another context is refused by on_lanes
    CUcontext ctx = nullptr;
    if (g_ctx_current(&ctx) != CUDA_SUCCESS || !ctx)
      return fail(FMX_ERR_CUDA, "no current CUDA context to create the lane objects in");
    if ((rc = make_lane_objects(c, ctx))) return rc;
  }
  for (int k = 0; k < kNumCounters; ++k) c->cap_c0[k] = *c->counter(k);
  c->cap_launches0 = c->launches;
  c->cap_fenced = c->fenced;
  c->cap_active = ++c->cap_next;
  return FMX_OK;
}

int fmx_graph_capture_end(fmx_comm_t c, void* graph, int* handle) {
  if (!c || !c->hdr || (graph && !handle)) return fail(FMX_ERR_INVALID_ARG, "null argument");
  if (!c->cap_active) return fail(FMX_ERR_INVALID_ARG, "no capture is active");
  c->cap_active = 0;
  c->fenced = c->cap_fenced;  // the captured calls did not run
  if (!graph) {  // the capture failed: abandon it (nothing was enqueued that will run)
    drop_pending(c);
    for (int k = 0; k < kNumCounters; ++k) *c->counter(k) = c->cap_c0[k];
    c->launches = c->cap_launches0;
    return FMX_OK;
  }
  if (c->pending) {  // a gather deferred inside the capture would never run
    drop_pending(c);
    for (int k = 0; k < kNumCounters; ++k) *c->counter(k) = c->cap_c0[k];
    c->launches = c->cap_launches0;
    return fail(FMX_ERR_INVALID_ARG, "the capture ended with a deferred gather: flush inside it");
  }
  CUgraph g = (CUgraph)graph;
  GraphRec rec;
  for (int k = 0; k < kNumCounters; ++k) {
    rec.c0[k] = c->cap_c0[k];
    rec.delta[k] = *c->counter(k) - c->cap_c0[k];
  }
  rec.launches = c->launches - c->cap_launches0;
  auto rollback = [&] {
    for (int k = 0; k < kNumCounters; ++k) *c->counter(k) = c->cap_c0[k];
    c->launches = c->cap_launches0;
  };
  if (!c->lane_ctx) {
    rollback();
    return fail(FMX_ERR_INVALID_ARG, "no collective was captured");
  }
  CtxPush push(c->lane_ctx);
  auto nodes_of = [&](std::vector<CUgraphNode>& v) -> int {
    size_t n = 0;
    if (g_graph_nodes(g, nullptr, &n) != CUDA_SUCCESS) return fail(FMX_ERR_CUDA, "cuGraphGetNodes failed");
    v.resize(n);
    if (n && g_graph_nodes(g, v.data(), &n) != CUDA_SUCCESS)
      return fail(FMX_ERR_CUDA, "cuGraphGetNodes failed");
    v.resize(n);
    return FMX_OK;
  };
  std::vector<CUgraphNode> nodes;
  int rc = nodes_of(nodes);
  // the end-of-replay fence, after every leaf of the captured graph
  if (rc == FMX_OK && c->nranks > 1) {
    std::vector<CUgraphNode> leaves;
    for (CUgraphNode nd : nodes) {
      size_t k = 0;
      if (g_node_dependents(nd, nullptr, &k) != CUDA_SUCCESS) {
        rc = fail(FMX_ERR_CUDA, "cuGraphNodeGetDependentNodes failed");
        break;
      }
      if (k == 0) leaves.push_back(nd);
    }
    const uint32_t v = c->fence_round + 1;
    CUstreamBatchMemOpParams sig;
    memset(&sig, 0, sizeof sig);
    sig.writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_32;
    sig.writeValue.address = c->flag_dev(c->rank, kFence);
    sig.writeValue.value = v;
    sig.writeValue.flags = CU_STREAM_WRITE_VALUE_DEFAULT;
    std::vector<CUstreamBatchMemOpParams> waits;
    for (int q = 0; q < c->nranks; ++q) {
      if (q == c->rank) continue;
      CUstreamBatchMemOpParams w;
      memset(&w, 0, sizeof w);
      w.waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_32;
      w.waitValue.address = c->flag_dev(q, kFence);
      w.waitValue.value = v;
      w.waitValue.flags = CU_STREAM_WAIT_VALUE_GEQ;
      waits.push_back(w);
    }
    CUDA_BATCH_MEM_OP_NODE_PARAMS p;
    memset(&p, 0, sizeof p);
    p.ctx = c->lane_ctx;
    p.count = 1;
    p.paramArray = &sig;
    CUgraphNode sn = nullptr, wn = nullptr;
    if (rc == FMX_OK && g_add_memop(&sn, g, leaves.data(), leaves.size(), &p) != CUDA_SUCCESS)
      rc = fail(FMX_ERR_CUDA, "adding the fence signal node failed");
    p.count = (unsigned)waits.size();
    p.paramArray = waits.data();
    if (rc == FMX_OK && g_add_memop(&wn, g, &sn, 1, &p) != CUDA_SUCCESS)
      rc = fail(FMX_ERR_CUDA, "adding the fence wait node failed");
    rec.delta[kCtrFence] += 1;
    if (rc == FMX_OK) rc = nodes_of(nodes);
  }
  // every memop node on this communicator's flags
  for (size_t i = 0; rc == FMX_OK && i < nodes.size(); ++i) {
    CUgraphNodeType t;
    if (g_node_type(nodes[i], &t) != CUDA_SUCCESS) {
      rc = fail(FMX_ERR_CUDA, "cuGraphNodeGetType failed");
      break;
    }
    if (t != CU_GRAPH_NODE_TYPE_BATCH_MEM_OP) continue;
    CUDA_BATCH_MEM_OP_NODE_PARAMS p;
    if (g_memop_get(nodes[i], &p) != CUDA_SUCCESS) {
      rc = fail(FMX_ERR_CUDA, "cuGraphBatchMemOpNodeGetParams failed");
      break;
    }
    GraphMemop m;
    m.node = nodes[i];
    m.ctx = p.ctx;
    m.flags = p.flags;
    m.ops.assign(p.paramArray, p.paramArray + p.count);
    bool mine = false;
    for (const CUstreamBatchMemOpParams& op : m.ops) {
      CUdeviceptr a = 0;
      if (op.operation == CU_STREAM_MEM_OP_WRITE_VALUE_32) a = op.writeValue.address;
      else if (op.operation == CU_STREAM_MEM_OP_WAIT_VALUE_32) a = op.waitValue.address;
      const int k = a ? flag_counter(c, a) : -1;
      if (k == -2) {
        rc = fail(FMX_ERR_UNSUPPORTED, "captured memop on an unexpected flag");
        break;
      }
      m.ctr.push_back((int8_t)k);
      mine |= k >= 0;
    }
    if (mine) rec.memops.push_back(std::move(m));
  }
  rollback();
  if (rc) return rc;
  c->graphs.push_back(std::move(rec));
  *handle = (int)c->graphs.size() - 1;
  return FMX_OK;
}

int fmx_graph_launch_prepare(fmx_comm_t c, int handle, void* graph_exec, void* stream) {
  int rc = check_comm(c);
  if (rc) return rc;
  if (handle < 0 || handle >= (int)c->graphs.size() || !c->graphs[handle].live || !graph_exec)
    return fail(FMX_ERR_INVALID_ARG, "bad graph handle");
  if (c->cap_active) return fail(FMX_ERR_INVALID_ARG, "launch_prepare inside a capture");
  GraphRec& rec = c->graphs[handle];
  cudaStream_t s = (cudaStream_t)stream;
  if (!c->fenced && c->nranks > 1) {
    // collectives ran since the last replay: fence first, on the launch stream
    cudaStream_t js = c->join_stream;
    c->join_stream = nullptr;
    rc = fmx_comm_fence(c, stream);
    c->join_stream = js;
    if (rc) return rc;
  }
  CtxPush push(c->lane_ctx);
  if (c->graph_stream && c->graph_stream != s) {  // previous replay on another stream
    FMX_CUDA(cudaEventRecord(c->graph_ev, c->graph_stream));
    FMX_CUDA(cudaStreamWaitEvent(s, c->graph_ev, 0));
  }
  if (c->has_done && c->done_cap == 0) FMX_CUDA(cudaStreamWaitEvent(s, c->done, 0));
  uint32_t off[kNumCounters];
  for (int k = 0; k < kNumCounters; ++k) off[k] = *c->counter(k) - rec.c0[k];
  if (rec.exec != (CUgraphExec)graph_exec || memcmp(off, rec.applied, sizeof off) != 0) {
    std::vector<CUstreamBatchMemOpParams> ops;
    for (const GraphMemop& m : rec.memops) {
      ops = m.ops;
      for (size_t i = 0; i < ops.size(); ++i) {
        if (m.ctr[i] < 0) continue;
        if (ops[i].operation == CU_STREAM_MEM_OP_WRITE_VALUE_32) ops[i].writeValue.value += off[m.ctr[i]];
        else ops[i].waitValue.value += off[m.ctr[i]];
      }
      CUDA_BATCH_MEM_OP_NODE_PARAMS p;
      memset(&p, 0, sizeof p);
      p.ctx = m.ctx;
      p.count = (unsigned)ops.size();
      p.paramArray = ops.data();
      p.flags = m.flags;
      CUresult r = g_exec_memop_set((CUgraphExec)graph_exec, m.node, &p);
      if (r != CUDA_SUCCESS) {
        rec.exec = nullptr;
        return fail(FMX_ERR_CUDA, "cuGraphExecBatchMemOpNodeSetParams failed (%d)", (int)r);
      }
    }
    rec.exec = (CUgraphExec)graph_exec;
    memcpy(rec.applied, off, sizeof off);
  }
  for (int k = 0; k < kNumCounters; ++k) *c->counter(k) += rec.delta[k];
  c->fenced = true;
  c->graph_stream = s;
  c->launches += rec.launches;
  return FMX_OK;
}

int fmx_graph_release(fmx_comm_t c, int handle) {
  if (!c || handle < 0 || handle >= (int)c->graphs.size())
    return fail(FMX_ERR_INVALID_ARG, "bad graph handle");
  c->graphs[handle].live = false;
  c->graphs[handle].memops.clear();
  c->graphs[handle].exec = nullptr;
  return FMX_OK;
}

int fmx_comm_kernel_launches(fmx_comm_t c, uint64_t* launches) {
  if (!c || !launches) return fail(FMX_ERR_INVALID_ARG, "null argument");
  *launches = c->launches;
  return FMX_OK;
}

}  // extern "C"

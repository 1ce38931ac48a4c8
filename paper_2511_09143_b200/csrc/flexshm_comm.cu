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
//    R % 2 of every region (double buffering).  Per round a rank (1) stages
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
//    MPS are time-sliced.  Slot reuse needs no credit messages: the waits of
//    round R already imply every peer finished round R-1.
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

#include "fmx_internal.h"
#include "flexshm_kernels.cuh"

using namespace fmx;

namespace {

typedef CUresult (*PFN_batchMemOp)(CUstream, unsigned int, CUstreamBatchMemOpParams*,
                                   unsigned int);
typedef CUresult (*PFN_streamGetCtx)(CUstream, CUcontext*);
typedef CUresult (*PFN_ctxPush)(CUcontext);
typedef CUresult (*PFN_ctxPop)(CUcontext*);
PFN_batchMemOp g_batch = nullptr;
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
  });
  if (g_driver_status != FMX_OK)
    return fail(FMX_ERR_UNSUPPORTED, "driver entry points (stream mem ops / contexts) unavailable");
  return FMX_OK;
}

#define FMX_CUDA(call)                                                                    \
  do {                                                                                    \
    cudaError_t _e = (call);                                                              \
    if (_e != cudaSuccess)                                                                \
      return fail(FMX_ERR_CUDA, "%s failed: %s (%s:%d)", #call, cudaGetErrorString(_e), \
                  __FILE__, __LINE__);                                                    \
  } while (0)

constexpr size_t kDefaultSliceCap = 4u << 20;   // bytes per (owner, contributor) slot
constexpr size_t kSegmentBudget = 1ull << 30;   // default cap on data-slot bytes
constexpr int kBatchMax = 128;                  // memops per cuStreamBatchMemOp call
constexpr int kNumEvents = 2 * FMX_MAX_SLOTS + 7;  // W[K], G[K]; host path F[2], C[2], inputs, P[2]

bool pid_alive(int pid) { return pid > 0 && (kill(pid, 0) == 0 || errno == EPERM); }

}  // namespace

struct fmx_comm;
static inline cudaStream_t lane_stream(const fmx_comm* c, int lane);

struct fmx_comm {
  int rank = -1, nranks = 0, nslots = 2, transport = FMX_TRANSPORT_CE, mig_aware = 1;
  size_t slice_bytes = 0, total_bytes = 0;
  Layout L{};
  char* base = nullptr;   // host VA of the mapping
  char* dbase = nullptr;  // device VA of the same bytes
  Header* hdr = nullptr;
  bool registered = false;
  uint32_t ar_round = 0, bc_round = 0;
  int64_t barrier_gen = 0;
  char* scratch = nullptr;  // CE transport: n * slice_bytes of HBM
  cudaStream_t lane[2] = {nullptr, nullptr};  // lane 0 (stage) and lane 2 (gather); lane 1 is the caller's stream
  cudaStream_t user = nullptr;                 // caller's stream of the current collective
  CUcontext lane_ctx = nullptr;                // context the lane objects were created in
  cudaEvent_t ev[kNumEvents] = {};  // intra-rank lane sync (see the kEv* ids)
  cudaEvent_t fork = nullptr, joined[2] = {nullptr, nullptr};
  bool result_via_ce = false;  // CE transport: result slot by copy engine, not SM stores
  bool copy2d = true;          // coalesce regular copy runs into cudaMemcpy2DAsync
  bool coarse = true;          // FMX_GRAIN=fine: per-piece waits instead of all-peer
  bool coarse_gather = true;   // FMX_GATHER_GRAIN=fine: per-owner gather waits only
  bool ramp = true;            // FMX_RAMP=0: equal rounds (no pipeline-fill ramp)
  int nlanes = 3;              // FMX_LANES=1: one stream; 2: gather on the reduce lane
  // live kernel timing (fmx_comm_set_timing): event pairs around every reduce
  bool timing = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> timed;
  size_t timed_used = 0;
  cudaEvent_t done = nullptr;
  bool has_done = false;
  uint64_t launches = 0;
  // pipeline timeline probe (fmx_comm_set_stamps): device ring of Stamp entries
  Stamp* stamps = nullptr;
  size_t stamp_cap = 0, stamp_used = 0;
  std::vector<fmx_peer_info> peers;
  std::vector<CUstreamBatchMemOpParams> ops;

  // byte offsets of the pipeline slots inside the segment
  size_t in_off(uint32_t R, int owner, int contrib) const {
    return L.ar_in_off + (((size_t)(R % nslots) * nranks + owner) * nranks + contrib) * slice_bytes;
  }
  size_t out_off(uint32_t R, int owner) const {
    return L.ar_out_off + ((size_t)(R % nslots) * nranks + owner) * slice_bytes;
  }
  size_t bc_slot_off(uint32_t R) const {
    return L.bc_off + (size_t)(R % nslots) * nranks * slice_bytes;
  }
  size_t user_region_off(int r) const { return L.user_off + (size_t)r * L.user_bytes; }
  // host (dev=false) or device (dev=true) address of a segment offset
  char* at(bool dev, size_t off) const { return (dev ? dbase : base) + off; }
  CUdeviceptr flag_dev(int r, int f) const {
    return (CUdeviceptr)(dbase + L.flags_off + ((size_t)r * kFlagsPerRank + f) * 64);
  }
  volatile uint32_t* flag_host(int r, int f) const {
    return (volatile uint32_t*)(base + L.flags_off + ((size_t)r * kFlagsPerRank + f) * 64);
  }
};

static inline cudaStream_t lane_stream(const fmx_comm* c, int lane) {
  if (c->nlanes == 1 || lane == 1) return c->user;
  if (lane == 0) return c->lane[0];
  return c->nlanes == 3 ? c->lane[1] : c->user;
}

namespace {

void unmap(fmx_comm* c) {
  if (c->base) munmap(c->base, c->total_bytes);
  c->base = nullptr;
  c->hdr = nullptr;
}

// ---- the plan: what one rank enqueues for one collective -----------------------
//
// plan_allreduce / plan_broadcast describe the schedule once, against a Sink.
// Work is issued on two lanes (CUDA streams) per rank so the two link
// directions overlap inside a rank: lane 0 stages (HBM -> SHM, D2H), lane 1
// fetches, reduces and gathers (SHM -> HBM, H2D).  Lanes fork from / join
// back into the caller's stream at every collective.  CudaSink turns the
// plan into stream operations; TraceSink records, per lane, every SHM and
// user-buffer byte range touched and every flag signalled / waited on, so the
// schedule of every rank of any world size can be model-checked on a CPU
// (fmx_trace_plan, tests/test_protocol_model.py).

constexpr int kLaneStage = 0;   // D2H lane
constexpr int kLaneMain = 1;    // fetch (H2D) + reduce lane: the caller's stream
constexpr int kLaneGather = 2;  // all-gather (H2D) lane

// One data-movement end for the trace: SHM byte range (relative to the
// segment) or user-buffer byte range (relative to the buffer start), plus the
// rank/round that (should have) written SHM bytes.
struct Annot {
  int64_t off = -1;
  size_t bytes = 0;
  int writer = -1;
  uint32_t round = 0;
  bool scratch = false;  // a range of the rank's HBM scratch, not of the user buffer
};

struct PlanSeg {
  const char* src;
  char* dst;
  size_t bytes;
  Annot shm;        // the SHM end of this segment
  bool shm_is_dst;  // true: this step writes SHM; false: reads it
  Annot user;       // the user-buffer end (off < 0: none, e.g. HBM scratch)
};

struct PlanReduce {
  ReduceArgs args;
  std::vector<Annot> reads;  // SHM inputs (ZC transport)
  Annot write;               // SHM result slot (written by the kernel)
  Annot user_rw;             // own piece of the user buffer (read + written)
  std::vector<Annot> scratch_reads;  // HBM scratch inputs (CE transport, host path)
  Annot scratch_write;               // HBM scratch result (host path)
  int dtype;
  bool aligned;
};

struct Sink {
  virtual ~Sink() {}
  virtual int copy(int lane, const std::vector<PlanSeg>& segs, bool src_sys, bool use_kernel) = 0;
  virtual int reduce(int lane, const PlanReduce& r) = 0;
  virtual int signal(int lane, int flag, uint32_t v) = 0;
  virtual int signal2(int lane, int f0, uint32_t v0, int f1, uint32_t v1) = 0;
  virtual int wait_peers(int lane, int flag, uint32_t v, int skip) = 0;
  virtual int wait_rank(int lane, int q, int flag, uint32_t v) = 0;
  virtual int d2d(int lane, void* dst, const void* src, size_t bytes, Annot from, Annot to) = 0;
  // intra-rank lane ordering through CUDA events (enqueue-order semantics)
  virtual int record(int lane, int ev) = 0;
  virtual int wait_event(int lane, int ev) = 0;
  // host-program accesses to SHM around a collective (trace only)
  virtual int host_access(int lane, const Annot& a, bool write) { return FMX_OK; }
};

int grid_for(size_t work_items, int threads, int cap) {
  size_t g = (work_items + threads - 1) / threads;
  return (int)std::max<size_t>(1, std::min<size_t>(g, (size_t)cap));
}

enum StampKind { kStWaitPeers = 1, kStWaitRank, kStWaitEvent, kStCopy, kStReduce, kStSignal };

class CudaSink final : public Sink {
 public:
  CudaSink(fmx_comm* c) : c_(c) {}

  // timeline probe: stamp the completion of the op just enqueued on `lane`
  int stamp(int lane, int kind, uint32_t info) {
    if (!c_->stamps || c_->stamp_used >= c_->stamp_cap) return FMX_OK;
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
    for (size_t i0 = 0; i0 < segs.size(); i0 += kMaxSegs) {
      CopyArgs a;
      memset(&a, 0, sizeof a);
      a.nseg = (int)std::min<size_t>(kMaxSegs, segs.size() - i0);
      a.src_sys = src_sys ? 1 : 0;
      size_t maxb = 0;
      for (int k = 0; k < a.nseg; ++k) {
        a.seg[k] = CopySeg{segs[i0 + k].src, segs[i0 + k].dst, segs[i0 + k].bytes};
        maxb = std::max(maxb, a.seg[k].bytes);
      }
      constexpr int kThreads = 512, kU = 4;
      int gx = grid_for((maxb / 16 + kU - 1) / kU, kThreads, std::max(1, 1184 / a.nseg));
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
    cudaStream_t s = lane_stream(c_, lane);
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    if (c_->timing) {
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
    constexpr int kThreads = 256, kU = 2;
    const int V = r.dtype == FMX_FLOAT32 ? 4 : 8;
    if (r.aligned) {
      int g = grid_for((a.len / V + kU - 1) / kU + 1, kThreads, 1184);
      if (r.dtype == FMX_FLOAT32)
        fmx_reduce_kernel<float, kU><<<g, kThreads, 0, s>>>(a);
      else
        fmx_reduce_kernel<__nv_bfloat16, kU><<<g, kThreads, 0, s>>>(a);
    } else {
      int g = grid_for(a.len, kThreads, 1184);
      if (r.dtype == FMX_FLOAT32)
        fmx_reduce_scalar_kernel<float><<<g, kThreads, 0, s>>>(a);
      else
        fmx_reduce_scalar_kernel<__nv_bfloat16><<<g, kThreads, 0, s>>>(a);
    }
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
    return FMX_OK;
  }

  int wait_event_impl(int lane, int ev) {
    FMX_CUDA(cudaStreamWaitEvent(lane_stream(c_, lane), c_->ev[ev], 0));
    return FMX_OK;
  }

  // every op, then (timeline probe on) a stamp of its completion on its lane
  int copy(int lane, const std::vector<PlanSeg>& segs, bool src_sys, bool use_kernel) override {
    size_t bytes = 0;
    for (const PlanSeg& g : segs) bytes += g.bytes;
    int rc = copy_impl(lane, segs, src_sys, use_kernel);
    return rc || segs.empty() ? rc : stamp(lane, kStCopy, (uint32_t)std::min<size_t>(bytes, ~0u));
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

// Text trace, one line per access / flag operation, prefixed by the lane:
//   <lane> W <off> <bytes> <round>           write SHM bytes of `round`
//   <lane> R <off> <bytes> <writer> <round>  read SHM bytes `writer` wrote in `round`
//   <lane> UR <off> <bytes> / UW <off> <bytes>   read / write own user buffer
//   <lane> S <flag> <value>                  signal own flag
//   <lane> A <rank> <flag> <value>           wait until rank's flag >= value
//   J                                        both lanes join (collective boundary)
class TraceSink final : public Sink {
 public:
  explicit TraceSink(std::string* out) : out_(out) {}
  int copy(int lane, const std::vector<PlanSeg>& segs, bool, bool) override {
    for (const PlanSeg& g : segs) {
      if (g.shm_is_dst) {
        user(lane, g.user, false);
        shm(lane, g.shm, true);
      } else {
        shm(lane, g.shm, false);
        user(lane, g.user, true);
      }
    }
    return FMX_OK;
  }
  int reduce(int lane, const PlanReduce& r) override {
    for (const Annot& a : r.reads) shm(lane, a, false);
    for (const Annot& a : r.scratch_reads) user(lane, a, false);
    user(lane, r.user_rw, false);
    user(lane, r.user_rw, true);
    user(lane, r.scratch_write, true);
    shm(lane, r.write, true);
    return FMX_OK;
  }
  int signal(int lane, int flag, uint32_t v) override { return line("%d S %d %u\n", lane, flag, v); }
  int signal2(int lane, int f0, uint32_t v0, int f1, uint32_t v1) override {
    line("%d S %d %u\n", lane, f0, v0);
    return line("%d S %d %u\n", lane, f1, v1);
  }
  int wait_peers(int lane, int flag, uint32_t v, int skip) override {
    for (int q = 0; q < nranks; ++q)
      if (q != skip) line("%d A %d %d %u\n", lane, q, flag, v);
    return FMX_OK;
  }
  int wait_rank(int lane, int q, int flag, uint32_t v) override {
    return line("%d A %d %d %u\n", lane, q, flag, v);
  }
  int d2d(int lane, void*, const void*, size_t, Annot from, Annot to) override {
    user(lane, from, false);
    user(lane, to, true);
    return FMX_OK;
  }
  int record(int lane, int ev) override { return line("%d E %d %d\n", lane, ev, ++seq_[ev]); }
  int wait_event(int lane, int ev) override {
    return seq_[ev] ? line("%d X %d %d\n", lane, ev, seq_[ev]) : FMX_OK;
  }
  int host_access(int lane, const Annot& a, bool write) override {
    shm(lane, a, write);
    return FMX_OK;
  }
  int join() { return line("J\n"); }
  int nranks = 0;

 private:
  void shm(int lane, const Annot& a, bool write) {
    if (a.off < 0 || a.bytes == 0) return;
    if (write)
      line("%d W %lld %zu %u\n", lane, (long long)a.off, a.bytes, a.round);
    else
      line("%d R %lld %zu %d %u\n", lane, (long long)a.off, a.bytes, a.writer, a.round);
  }
  void user(int lane, const Annot& a, bool write) {
    if (a.off < 0 || a.bytes == 0) return;
    const char* kind = a.scratch ? (write ? "SW" : "SR") : (write ? "UW" : "UR");
    line("%d %s %lld %zu\n", lane, kind, (long long)a.off, a.bytes);
  }
  int line(const char* fmt, ...) __attribute__((format(printf, 2, 3))) {
    char buf[128];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    out_->append(buf);
    return FMX_OK;
  }
  std::string* out_;
  int seq_[kNumEvents] = {};
};

// Round j of every chunk covers [prefix(j), prefix(j) + size(j)).  With the
// ramp, the first rounds are slice/8, /4, /2 and the last ones /2, /4, /8: the
// pipeline fills (round 0's stage is pure D2H, the H2D direction idle) and
// drains (the last gather is pure H2D) in 1/8 of the time a full slice takes.
struct Geometry {
  size_t count, esz, chunk, slice;
  uint32_t rounds;
  std::vector<size_t> start;  // start[j] = prefix of round j; start[rounds] >= chunk
  size_t size(uint32_t j) const { return start[j + 1] - start[j]; }
  size_t lo(int owner, uint32_t j) const { return (size_t)owner * chunk + start[j]; }
  size_t len(int owner, uint32_t j) const {
    size_t a = lo(owner, j);
    size_t end = std::min((size_t)(owner + 1) * chunk, count);
    if (a >= end) return 0;
    return std::min(size(j), end - a);
  }
};

// chunk_elems = 0: allreduce chunking (16-byte aligned chunk starts over
// `count`); otherwise every rank's chunk has exactly chunk_elems elements and
// count = n * chunk_elems (reduce-scatter / all-gather, NCCL's layout).
Geometry allreduce_geometry(const fmx_comm* c, size_t count, int dtype, size_t chunk_elems = 0) {
  Geometry g;
  const int n = c->nranks;
  g.esz = dtype == FMX_FLOAT32 ? 4 : 2;
  const size_t vec = 16 / g.esz;
  g.count = chunk_elems ? chunk_elems * n : count;
  g.chunk = chunk_elems ? chunk_elems : ((count + n - 1) / n + vec - 1) / vec * vec;
  g.slice = c->slice_bytes / g.esz;
  std::vector<size_t> sizes;
  const size_t s = g.slice;
  if (c->ramp && g.chunk > s) {
    // geometric ramp s/8, s/4, s/2 up and down (as much of it as fits in half
    // the chunk each way), the middle in equal rounds of at most s
    std::vector<size_t> up;
    size_t ramp_sum = 0;
    for (size_t x = s / 8; x < s && x > 0; x *= 2) {
      if (2 * (ramp_sum + x) > g.chunk) break;
      up.push_back(x);
      ramp_sum += x;
    }
    const size_t mid = g.chunk - 2 * ramp_sum;
    const size_t k = (mid + s - 1) / s;
    sizes = up;
    for (size_t i = 0; i < k; ++i) {  // equal split, multiples of the vector width
      const size_t lo = (mid * i / k) / vec * vec, hi = i + 1 == k ? mid : (mid * (i + 1) / k) / vec * vec;
      if (hi > lo) sizes.push_back(hi - lo);
    }
    sizes.insert(sizes.end(), up.rbegin(), up.rend());
  } else {
    for (size_t left = g.chunk; left;) {
      const size_t y = std::min(s, left);
      sizes.push_back(y);
      left -= y;
    }
  }
  if (sizes.empty()) sizes.push_back(0);  // count == 0 never reaches here; keep rounds >= 1
  g.rounds = (uint32_t)sizes.size();
  g.start.assign(g.rounds + 1, 0);
  for (uint32_t j = 0; j < g.rounds; ++j) g.start[j + 1] = g.start[j] + sizes[j];
  return g;
}

Annot ubuf(size_t off_bytes, size_t bytes) { return Annot{(int64_t)off_bytes, bytes, -1, 0}; }
Annot sbuf(size_t off_bytes, size_t bytes) { return Annot{(int64_t)off_bytes, bytes, -1, 0, true}; }

// Reduce-scatter + all-gather through the segment, pipelined in rounds on three
// lanes: lane 0 stages (D2H), lane 1 fetches and reduces (H2D + kernel), lane 2
// gathers (H2D).  Round R uses slot R % 2.  With the gather on its own lane, a
// rank fetches round R+1 while it still waits for the slowest owner of round R,
// so the H2D direction never idles at a round boundary.
//
// Enqueue order is itself a valid single-stream schedule: every wait (flag or
// event) points at work enqueued earlier, by this rank or by peers that enqueue
// in the same order.  So however the driver maps the lane streams onto
// hardware queues - even one shared FIFO - nothing can deadlock; separate queues
// only add overlap.  Lane 0 never waits on a flag: only on events of lane 2.
// The model checker checks both the multi-lane and the merged single-FIFO reading.
//
// Events (slot = round parity): W(R) is recorded on the gather lane once every
// peer's REDUCED >= R+1 was seen, G(R) once gather(R) completed.  REDUCED(R)
// (value R+1) is signalled after reduce(R) AND G(R-1), so "REDUCED[q] >= R+1"
// also says "q finished gathering round R-1".
//
// Hazards and the wait that covers each:
//  stage(R) into in[R%2][o][me], last read by owner o's fetch of round R-2:
//      W(R-2) (every owner signalled REDUCED after its fetches of R-2); rounds
//      of an earlier collective are covered by the fork.
//  fetch(R) of in[R%2][me][q]              -> wait STAGED(_TO)[q] >= R+1
//  reduce(R) writes out[R%2][me], last read by every q's gather(R-2):
//      W(R-1): every q signalled REDUCED >= R, which q issued after G_q(R-2).
//  gather(R) reads out[R%2][q]             -> wait REDUCED[q] >= R+1
//  in place: gather(R) overwrites piece (q, R); my stage(R) read it first,
//      because owner q's reduce(R) waited for my STAGED >= R+1.
// With FMX_LANES=2 the gather runs on lane 1 and the W/G waits are implied by
// stream order (the schedule of the first B200 runs).
enum { kEvSlotFree = 0, kEvGathered = FMX_MAX_SLOTS };  // + R % K: W(R) and G(R) above

// The three owner-chunk collectives share one schedule:
//   kAllreduce     stage -> fetch -> reduce (HBM + result slot) -> gather
//   kReduceScatter stage -> fetch -> reduce into recv (no result slot, no gather copies)
//   kAllgather     publish my chunk (result slot + my part of recv) -> gather
// Flags, events and slot reuse are identical, so one model-checked protocol
// covers all three.  For the last two, `count` is the per-rank count and the
// buffers follow NCCL: send/recv of reduce-scatter hold n*count / count
// elements, those of all-gather count / n*count.
enum Kind { kAllreduce = 0, kReduceScatter = 1, kAllgather = 2 };

int plan_allreduce(fmx_comm* c, Sink& k, const char* src, char* dst, size_t count, int dtype,
                   int op, float factor, bool aligned, int kind = kAllreduce) {
  const int n = c->nranks, me = c->rank;
  const bool zc = c->transport == FMX_TRANSPORT_ZC;
  const int LG = c->nlanes == 3 ? kLaneGather : kLaneMain;
  const int K = c->nslots;  // pipeline depth: slots per region
  const bool split = LG != kLaneMain;  // gather on its own lane: explicit W / G waits
  const bool ar = kind == kAllreduce, rs = kind == kReduceScatter, ag = kind == kAllgather;
  const Geometry g = allreduce_geometry(c, count, dtype, ar ? 0 : count);
  // where piece (me, j) of the result goes, and where my contribution / my
  // published chunk comes from (all-gather's send holds only my chunk)
  auto my_out = [&](uint32_t j) { return dst + (rs ? g.start[j] : g.lo(me, j)) * g.esz; };
  auto my_in = [&](uint32_t j) { return src + (ag ? g.start[j] : g.lo(me, j)) * g.esz; };
  std::vector<PlanSeg> segs;
  int rc;
  const uint32_t R0 = c->ar_round;
  // peers in rotated order starting after me, so that at any moment the
  // ranks work on different owners / contributors instead of all on one
  auto rot = [&](int i) { return (me + 1 + i) % n; };

  auto stage = [&](uint32_t j) -> int {
    const uint32_t R = R0 + j;
    if (ag) return FMX_OK;  // nothing to reduce: no contributions to stage
    // slot R%K was read by round R-K's fetches: W(R-K)
    if (j >= K && (rc = k.wait_event(kLaneStage, kEvSlotFree + R % K))) return rc;
    if (c->coarse) {  // one batch of copies, one STAGED signal
      segs.clear();
      for (int o = 0; o < n; ++o) {
        const size_t len = o == me ? 0 : g.len(o, j);
        if (!len) continue;
        const size_t off = c->in_off(R, o, me);
        segs.push_back({src + g.lo(o, j) * g.esz, c->at(zc, off), len * g.esz,
                        Annot{(int64_t)off, len * g.esz, me, R}, true,
                        ubuf(g.lo(o, j) * g.esz, len * g.esz)});
      }
      if ((rc = k.copy(kLaneStage, segs, false, zc))) return rc;
      return k.signal(kLaneStage, kStaged, R + 1);
    }
    for (int i = 0; i < n - 1; ++i) {
      const int o = rot(i);
      const size_t len = g.len(o, j);
      segs.clear();
      if (len) {
        const size_t off = c->in_off(R, o, me);
        segs.push_back({src + g.lo(o, j) * g.esz, c->at(zc, off), len * g.esz,
                        Annot{(int64_t)off, len * g.esz, me, R}, true,
                        ubuf(g.lo(o, j) * g.esz, len * g.esz)});
        if ((rc = k.copy(kLaneStage, segs, false, zc))) return rc;
      }
      if ((rc = k.signal(kLaneStage, kStagedTo + o, R + 1))) return rc;
    }
    return FMX_OK;
  };

  // lane 0 stages K-1 rounds ahead of the reduction
  const uint32_t ahead = (uint32_t)K - 1;
  for (uint32_t j = 0; j < ahead && j < g.rounds; ++j)
    if ((rc = stage(j))) return rc;
  for (uint32_t j = 0; j < g.rounds; ++j) {
    const uint32_t R = R0 + j;
    if (j + ahead < g.rounds && (rc = stage(j + ahead))) return rc;
    // lane 1: fetch, then reduce-scatter my chunk in ascending rank order
    const size_t mylen = g.len(me, j);
    if (mylen && ag) {
      // publish: my piece into my result slot (and into my part of recv)
      const size_t out_off = c->out_off(R, me);
      if (split && j + 1 >= K && (rc = k.wait_event(kLaneMain, kEvSlotFree + (R + 1 - K) % K)))
        return rc;
      segs.clear();
      segs.push_back({my_in(j), c->at(zc, out_off), mylen * g.esz,
                      Annot{(int64_t)out_off, mylen * g.esz, me, R}, true,
                      ubuf(g.lo(me, j) * g.esz, mylen * g.esz)});
      if ((rc = k.copy(kLaneMain, segs, false, zc))) return rc;
      if (my_out(j) != my_in(j) &&
          (rc = k.d2d(kLaneMain, my_out(j), my_in(j), mylen * g.esz,
                      ubuf(g.lo(me, j) * g.esz, mylen * g.esz),
                      ubuf(g.lo(me, j) * g.esz, mylen * g.esz))))
        return rc;
    } else if (mylen) {
      PlanReduce pr;
      memset(&pr.args, 0, sizeof pr.args);
      pr.dtype = dtype;
      pr.aligned = aligned;
      ReduceArgs& a = pr.args;
      a.nsrc = n;
      a.len = mylen;
      a.op = op;
      a.factor = factor;
      a.out_dev = my_out(j);
      const size_t out_off = c->out_off(R, me);
      pr.user_rw = ubuf(g.lo(me, j) * g.esz, mylen * g.esz);
      const bool via_ce = ar && !zc && c->result_via_ce;
      if (ar && !via_ce) {
        a.out_sys = c->at(true, out_off);
        pr.write = Annot{(int64_t)out_off, mylen * g.esz, me, R};
      }
      // each contribution is fetched as soon as its contributor staged it
      if (c->coarse) {
        if ((rc = k.wait_peers(kLaneMain, kStaged, R + 1, me))) return rc;
        if (!zc) {
          segs.clear();
          for (int q = 0; q < n; ++q) {
            if (q == me) continue;
            const size_t off = c->in_off(R, me, q);
            segs.push_back({c->at(false, off), c->scratch + (size_t)q * c->slice_bytes,
                            mylen * g.esz, Annot{(int64_t)off, mylen * g.esz, q, R}, false,
                            sbuf((size_t)q * c->slice_bytes, mylen * g.esz)});
          }
          if ((rc = k.copy(kLaneMain, segs, true, false))) return rc;
        }
      }
      for (int i = 0; i < n - 1 && !c->coarse; ++i) {
        const int q = rot(i);
        if ((rc = k.wait_rank(kLaneMain, q, kStagedTo + me, R + 1))) return rc;
        if (!zc) {
          const size_t off = c->in_off(R, me, q);
          segs.clear();
          segs.push_back({c->at(false, off), c->scratch + (size_t)q * c->slice_bytes,
                          mylen * g.esz, Annot{(int64_t)off, mylen * g.esz, q, R}, false,
                          sbuf((size_t)q * c->slice_bytes, mylen * g.esz)});
          if ((rc = k.copy(kLaneMain, segs, true, false))) return rc;
        }
      }
      for (int q = 0; q < n; ++q) {
        if (q == me) {
          a.src[q] = my_in(j);
        } else if (zc) {
          const size_t off = c->in_off(R, me, q);
          a.src[q] = c->at(true, off);
          a.sys_mask |= 1ull << q;
          pr.reads.push_back(Annot{(int64_t)off, mylen * g.esz, q, R});
        } else {
          a.src[q] = c->scratch + (size_t)q * c->slice_bytes;
          pr.scratch_reads.push_back(sbuf((size_t)q * c->slice_bytes, mylen * g.esz));
        }
      }
      // out[R%K][me] is free once every peer gathered round R-K: W(R-K+1)
      if (split && j + 1 >= K && (rc = k.wait_event(kLaneMain, kEvSlotFree + (R + 1 - K) % K)))
        return rc;
      if ((rc = k.reduce(kLaneMain, pr))) return rc;
      if (via_ce) {  // result slot written by the copy engine from HBM
        segs.clear();
        segs.push_back({my_out(j), c->at(false, out_off), mylen * g.esz,
                        Annot{(int64_t)out_off, mylen * g.esz, me, R}, true,
                        ubuf(g.lo(me, j) * g.esz, mylen * g.esz)});
        if ((rc = k.copy(kLaneMain, segs, false, false))) return rc;
      }
    }
    // REDUCED(R) also says "my gather(R-1) is done": G(R-1)
    if (split && j >= 1 && (rc = k.wait_event(kLaneMain, kEvGathered + (R - 1) % K))) return rc;
    if ((rc = k.signal(kLaneMain, kReduced, R + 1))) return rc;
    // all-gather (lane LG): each owner's result as soon as that owner has it
    if (c->coarse_gather) {
      if ((rc = k.wait_peers(LG, kReduced, R + 1, me))) return rc;
      if ((rc = k.record(LG, kEvSlotFree + R % K))) return rc;  // W(R)
      segs.clear();
      for (int q = 0; q < n && !rs; ++q) {
        const size_t len = q == me ? 0 : g.len(q, j);
        if (!len) continue;
        const size_t off = c->out_off(R, q);
        segs.push_back({c->at(zc, off), dst + g.lo(q, j) * g.esz, len * g.esz,
                        Annot{(int64_t)off, len * g.esz, q, R}, false,
                        ubuf(g.lo(q, j) * g.esz, len * g.esz)});
      }
      if ((rc = k.copy(LG, segs, true, zc))) return rc;
    } else {
      for (int i = 0; i < n - 1; ++i) {
        const int q = rot(i);
        if ((rc = k.wait_rank(LG, q, kReduced, R + 1))) return rc;
        const size_t len = rs ? 0 : g.len(q, j);
        if (!len) continue;
        const size_t off = c->out_off(R, q);
        segs.clear();
        segs.push_back({c->at(zc, off), dst + g.lo(q, j) * g.esz, len * g.esz,
                        Annot{(int64_t)off, len * g.esz, q, R}, false,
                        ubuf(g.lo(q, j) * g.esz, len * g.esz)});
        if ((rc = k.copy(LG, segs, true, zc))) return rc;
      }
      if ((rc = k.record(LG, kEvSlotFree + R % K))) return rc;  // W(R)
    }
    if (split && (rc = k.record(LG, kEvGathered + R % K))) return rc;  // G(R)
  }
  c->ar_round += g.rounds;
  return FMX_OK;
}

// Allreduce over the ranks' registered host buffers (the regions at the end of
// the segment): in place, no staging and no all-gather.  Every input already
// sits in host memory, so owner r copy-engines piece j of chunk r out of all n
// regions into HBM scratch (lane 0), reduces it in rank order (lane 1) and
// copy-engines the result into piece j of chunk r of every region (lane 1).
// Per GPU that is k*S H2D + k*S D2H, against 2k(n-1)/n*S + k*S (+ the
// caller's own k*S in and k*S out) for device buffers.
constexpr uint32_t kInputTag = 1u << 31;  // trace: "input written by the host for round R"
enum { kEvFetched = 2 * FMX_MAX_SLOTS, kEvConsumed = kEvFetched + 2, kEvInputs = kEvFetched + 4,
       kEvPushed = kEvFetched + 5 };

int plan_allreduce_host(fmx_comm* c, Sink& k, size_t off_bytes, size_t count, int dtype, int op,
                        float factor) {
  const int n = c->nranks, me = c->rank;
  const Geometry g = allreduce_geometry(c, count, dtype);
  const uint32_t R0 = c->ar_round, P = g.rounds;
  const size_t sb = c->slice_bytes;
  const int LP = c->nlanes == 3 ? kLaneGather : kLaneMain;  // push lane
  auto region = [&](int q, int o, uint32_t j) {
    return c->user_region_off(q) + off_bytes + g.lo(o, j) * g.esz;
  };
  std::vector<PlanSeg> segs;
  int rc;
  // the caller wrote its whole input before the call (host program order)
  for (int o = 0; o < n; ++o)
    for (uint32_t j = 0; j < P; ++j)
      if (size_t len = g.len(o, j))
        k.host_access(kLaneMain, Annot{(int64_t)region(me, o, j), len * g.esz, me,
                                       (R0 + j) | kInputTag}, true);
  // every rank's inputs are in place: exchange STAGED on lane 1, release lane 0
  if ((rc = k.signal(kLaneMain, kStaged, R0 + P))) return rc;
  if ((rc = k.wait_peers(kLaneMain, kStaged, R0 + P, me))) return rc;
  if ((rc = k.record(kLaneMain, kEvInputs))) return rc;
  if ((rc = k.wait_event(kLaneStage, kEvInputs))) return rc;
  for (uint32_t j = 0; j < P; ++j) {
    const uint32_t R = R0 + j, slot = j % 2;
    const size_t len = g.len(me, j);
    // scratch: fetch slots [2][n], result replicas [2][n] (one per region, so
    // the push is one 2D copy)
    const size_t fetch_off = (size_t)slot * n * sb, result_off = ((size_t)2 * n + slot * n) * sb;
    char* fetch = c->scratch + fetch_off;
    char* result = c->scratch + result_off;
    // lane 0: pull piece j of my chunk out of every region; the fetch slot is
    // free once lane 1's reduce of round j-2 consumed it (C(j-2)), so fetches
    // run up to two rounds ahead of the pushes
    if (j >= 2 && (rc = k.wait_event(kLaneStage, kEvConsumed + slot))) return rc;
    segs.clear();
    for (int q = 0; q < n && len; ++q) {
      const size_t off = region(q, me, j);
      segs.push_back({c->at(false, off), fetch + (size_t)q * sb, len * g.esz,
                      Annot{(int64_t)off, len * g.esz, q, R | kInputTag}, false,
                      sbuf(fetch_off + (size_t)q * sb, len * g.esz)});
    }
    if ((rc = k.copy(kLaneStage, segs, true, false))) return rc;
    if ((rc = k.record(kLaneStage, kEvFetched + slot))) return rc;
    // lane 1: reduce in rank order; the result slot j%2 is free once lane LP
    // pushed round j-2 (P(j-2))
    if ((rc = k.wait_event(kLaneMain, kEvFetched + slot))) return rc;
    if (j >= 2 && LP != kLaneMain && (rc = k.wait_event(kLaneMain, kEvPushed + slot))) return rc;
    if (len) {
      PlanReduce pr;
      memset(&pr.args, 0, sizeof pr.args);
      pr.dtype = dtype;
      pr.aligned = true;
      pr.args.nsrc = n;
      pr.args.len = len;
      pr.args.op = op;
      pr.args.factor = factor;
      pr.args.out_dev = result;
      pr.args.n_rep = n;
      pr.args.rep_stride = sb;
      for (int q = 0; q < n; ++q) {
        pr.args.src[q] = fetch + (size_t)q * sb;
        pr.scratch_reads.push_back(sbuf(fetch_off + (size_t)q * sb, len * g.esz));
      }
      pr.scratch_write = sbuf(result_off, n * sb);
      if ((rc = k.reduce(kLaneMain, pr))) return rc;
    }
    if ((rc = k.record(kLaneMain, kEvConsumed + slot))) return rc;  // C(j)
    // lane LP: push the result into every region, off the reduce lane so the
    // D2H direction never waits behind the next round's fetch
    if (LP != kLaneMain && (rc = k.wait_event(LP, kEvConsumed + slot))) return rc;
    if (len) {
      segs.clear();
      for (int q = 0; q < n; ++q) {
        const size_t off = region(q, me, j);
        segs.push_back({result + (size_t)q * sb, c->at(false, off), len * g.esz,
                        Annot{(int64_t)off, len * g.esz, me, R}, true,
                        sbuf(result_off, n * sb)});
      }
      if ((rc = k.copy(LP, segs, false, false))) return rc;
    }
    if (LP != kLaneMain && (rc = k.record(LP, kEvPushed + slot))) return rc;  // P(j)
  }
  if ((rc = k.signal(LP, kReduced, R0 + P))) return rc;
  if ((rc = k.wait_peers(LP, kReduced, R0 + P, me))) return rc;
  // the caller then reads its whole region (host program order)
  for (int o = 0; o < n; ++o)
    for (uint32_t j = 0; j < P; ++j)
      if (size_t len = g.len(o, j))
        k.host_access(LP, Annot{(int64_t)region(me, o, j), len * g.esz, o, R0 + j}, false);
  c->ar_round += P;
  return FMX_OK;
}

// Root stages rounds of n*slice bytes into the broadcast slot; every other
// rank copies them out and signals BC_DONE, which the root waits on before
// reusing a slot (two rounds later).  Single lane (lane 1).
int plan_broadcast(fmx_comm* c, Sink& k, const char* src, char* dst, size_t count, int dtype,
                   int root) {
  const int me = c->rank;
  const int L = kLaneMain;
  const bool zc = c->transport == FMX_TRANSPORT_ZC;
  const size_t esz = dtype == FMX_FLOAT32 ? 4 : 2;
  const size_t bslice = (size_t)c->nranks * c->slice_bytes / esz;
  const uint32_t rounds = (uint32_t)((count + bslice - 1) / bslice);
  std::vector<PlanSeg> segs(1);
  int rc;
  for (uint32_t j = 0; j < rounds; ++j) {
    const uint32_t R = c->bc_round + j;
    const size_t lo = (size_t)j * bslice, len = std::min(bslice, count - lo);
    const size_t off = c->bc_slot_off(R);
    const Annot an{(int64_t)off, len * esz, root, R};
    if (me == root) {
      if (R + 1 > (uint32_t)c->nslots && (rc = k.wait_peers(L, kBcDone, R + 1 - c->nslots, me)))
        return rc;
      segs[0] = {src + lo * esz, c->at(zc, off), len * esz, an, true, ubuf(lo * esz, len * esz)};
      if ((rc = k.copy(L, segs, false, zc))) return rc;
      if ((rc = k.signal2(L, kBcStaged, R + 1, kBcDone, R + 1))) return rc;
      if (src != dst &&
          (rc = k.d2d(L, dst + lo * esz, src + lo * esz, len * esz, Annot{}, Annot{})))
        return rc;
    } else {
      if ((rc = k.wait_rank(L, root, kBcStaged, R + 1))) return rc;
      segs[0] = {c->at(zc, off), dst + lo * esz, len * esz, an, false, ubuf(lo * esz, len * esz)};
      if ((rc = k.copy(L, segs, true, zc))) return rc;
      if ((rc = k.signal(L, kBcDone, R + 1))) return rc;
    }
  }
  c->bc_round += rounds;
  return FMX_OK;
}

// Fork the lanes off the caller's stream, run the plan, join them back.
// (Re)create the lane-0 stream and the lane events in `ctx`, the context of
// the caller's stream (a green context, an MPS client's, or the primary one),
// so every lane object lives where the caller's work lives.
int make_lane_objects(fmx_comm* c, CUcontext ctx) {
  c->lane[0] = c->lane[1] = nullptr;  // objects of an earlier context are abandoned, not destroyed
  for (int l = 0; l < 2; ++l) {
    FMX_CUDA(cudaStreamCreateWithFlags(&c->lane[l], cudaStreamNonBlocking));
    FMX_CUDA(cudaEventCreateWithFlags(&c->joined[l], cudaEventDisableTiming));
  }
  FMX_CUDA(cudaEventCreateWithFlags(&c->fork, cudaEventDisableTiming));
  FMX_CUDA(cudaEventCreateWithFlags(&c->done, cudaEventDisableTiming));
  for (int i = 0; i < kNumEvents; ++i) FMX_CUDA(cudaEventCreateWithFlags(&c->ev[i], cudaEventDisableTiming));
  for (auto& pr : c->timed) pr = {nullptr, nullptr};
  c->timed.clear();
  c->timed_used = 0;
  c->lane_ctx = ctx;
  return FMX_OK;
}

// Run one collective: lane 1 is the caller's stream, lane 0 forks off it and
// joins back.  Every runtime call happens with the caller's stream context
// current (DDP calls hooks from autograd threads whose current context may be
// another one).
template <typename F>
int on_lanes(fmx_comm* c, cudaStream_t user, F&& body) {
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
  if (ctx != c->lane_ctx && (rc = make_lane_objects(c, ctx))) return rc;
  c->user = user;
  const int forked = c->nlanes - 1;  // lane 0, then lane 2 (lane 1 is `user`)
  if (forked > 0) FMX_CUDA(cudaEventRecord(c->fork, user));
  for (int l = 0; l < forked; ++l) FMX_CUDA(cudaStreamWaitEvent(c->lane[l], c->fork, 0));
  rc = body();
  for (int l = 0; l < forked; ++l) {
    FMX_CUDA(cudaEventRecord(c->joined[l], c->lane[l]));
    FMX_CUDA(cudaStreamWaitEvent(user, c->joined[l], 0));
  }
  if (rc) return rc;
  FMX_CUDA(cudaEventRecord(c->done, user));
  c->has_done = true;
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
    nslots = 2;
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
      sb = std::min(kDefaultSliceCap, kSegmentBudget / per);
    }
    sb = std::max<size_t>(4096, sb / 4096 * 4096);
    Layout L = compute_layout(nranks, c->nslots, sb, host_bytes);
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
    h->user_off = L.user_off;
    h->user_bytes = L.user_bytes;
    h->creator_pid = (int32_t)getpid();
    h->mig_aware = mig_aware ? 1 : 0;
    snprintf(h->job_key, sizeof h->job_key, "%s", job_key);
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
          h->total_bytes != (uint64_t)st.st_size) {
        munmap(p, (size_t)st.st_size);
        usleep(1000);
        continue;
      }
      if (h->nranks != nranks) {
        munmap(p, (size_t)st.st_size);
        delete c;
        return fail(FMX_ERR_BAD_RANKS, "segment %s has %d ranks, caller says %d", name.c_str(),
                    h->nranks, nranks);
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
                h->user_off, h->user_bytes, h->total_bytes};
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
  if (rc != FMX_OK) {
    unmap(c);
    delete c;
    return rc;  // message / dup pair already set
  }

  c->transport = transport == FMX_TRANSPORT_AUTO ? FMX_TRANSPORT_CE : transport;
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


  if (const char* v = getenv("FMX_RESULT_VIA_CE")) c->result_via_ce = atoi(v) != 0;
  if (const char* v = getenv("FMX_COPY2D")) c->copy2d = atoi(v) != 0;
  if (const char* v = getenv("FMX_GRAIN")) c->coarse = strcmp(v, "fine") != 0;
  c->coarse_gather = c->coarse;
  if (const char* v = getenv("FMX_GATHER_GRAIN")) c->coarse_gather = strcmp(v, "fine") != 0;
  if (const char* v = getenv("FMX_LANES")) c->nlanes = std::min(3, std::max(1, atoi(v)));
  if (const char* v = getenv("FMX_RAMP")) c->ramp = atoi(v) != 0;
  if (e != cudaSuccess) {
    h->aborted.store(1);
    fail(FMX_ERR_CUDA, "device mapping of %zu-byte segment failed: %s", c->total_bytes,
         cudaGetErrorString(e));
    if (c->registered) cudaHostUnregister(c->base);
    if (c->scratch) cudaFree(c->scratch);
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
  if (op < FMX_OP_SUM || op > FMX_OP_PREDIV_SUM) return fail(FMX_ERR_INVALID_ARG, "bad op %d", op);
  if (op != FMX_OP_SUM && !std::isfinite(factor))
    return fail(FMX_ERR_INVALID_ARG, "factor must be finite");
  if (count == 0) return FMX_OK;
  if (!send || !recv) return fail(FMX_ERR_INVALID_ARG, "null buffer");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t esz = dtype == FMX_FLOAT32 ? 4 : 2;
  const bool aligned = (((uintptr_t)send | (uintptr_t)recv) & 15) == 0;
  CudaSink sink(c);
  if (c->nranks == 1) {  // nothing to exchange: apply the scale convention locally
    return on_lanes(c, s, [&]() -> int {
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
  return on_lanes(c, s, [&]() {
    return plan_allreduce(c, sink, (const char*)send, (char*)recv, count, dtype, op, factor,
                          aligned);
  });
}

// Shared argument checks of the dtype / op / factor triple.
static int check_reduction_args(int dtype, int op, float factor) {
  if (dtype != FMX_FLOAT32 && dtype != FMX_BFLOAT16)
    return fail(FMX_ERR_INVALID_ARG, "bad dtype %d", dtype);
  if (op < FMX_OP_SUM || op > FMX_OP_PREDIV_SUM) return fail(FMX_ERR_INVALID_ARG, "bad op %d", op);
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
  return on_lanes(c, (cudaStream_t)stream, [&]() -> int {
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
  return on_lanes(c, (cudaStream_t)stream, [&]() -> int {
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
  if (op < FMX_OP_SUM || op > FMX_OP_PREDIV_SUM) return fail(FMX_ERR_INVALID_ARG, "bad op %d", op);
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
  cudaStream_t s = (cudaStream_t)stream;
  constexpr int kThreads = 256, kU = 2;
  const int V = dtype == FMX_FLOAT32 ? 4 : 8;
  if ((bits & 15) == 0) {
    int g = grid_for((count / V + kU - 1) / kU + 1, kThreads, 1184);
    if (dtype == FMX_FLOAT32)
      fmx_reduce_kernel<float, kU><<<g, kThreads, 0, s>>>(a);
    else
      fmx_reduce_kernel<__nv_bfloat16, kU><<<g, kThreads, 0, s>>>(a);
  } else {
    int g = grid_for(count, kThreads, 1184);
    if (dtype == FMX_FLOAT32)
      fmx_reduce_scalar_kernel<float><<<g, kThreads, 0, s>>>(a);
    else
      fmx_reduce_scalar_kernel<__nv_bfloat16><<<g, kThreads, 0, s>>>(a);
  }
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
  if (op < FMX_OP_SUM || op > FMX_OP_PREDIV_SUM) return fail(FMX_ERR_INVALID_ARG, "bad op %d", op);
  if (op != FMX_OP_SUM && !std::isfinite(factor))
    return fail(FMX_ERR_INVALID_ARG, "factor must be finite");
  const size_t esz = dtype == FMX_FLOAT32 ? 4 : 2;
  if (offset % 16 || offset + count * esz > c->L.user_bytes)
    return fail(FMX_ERR_INVALID_ARG, "host range [%zu, +%zu) outside the %zu-byte region (16-B aligned offset required)",
                offset, count * esz, (size_t)c->L.user_bytes);
  if (count == 0) return FMX_OK;
  CudaSink sink(c);
  return on_lanes(c, (cudaStream_t)stream, [&]() {
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
    return on_lanes(c, s, [&]() -> int {
      if (send != recv)
        FMX_CUDA(cudaMemcpyAsync(recv, send, count * esz, cudaMemcpyDeviceToDevice, lane_stream(c, kLaneMain)));
      return FMX_OK;
    });
  }
  return on_lanes(c, s, [&]() {
    return plan_broadcast(c, sink, (const char*)send, (char*)recv, count, dtype, root);
  });
}

int fmx_trace_plan(int nranks, int rank, int transport, size_t slice_bytes, int nops,
                   const int* kinds, const size_t* counts, const int* dtypes, const int* roots,
                   char* buf, size_t cap, size_t* used) {
  if (nranks < 2 || nranks > FMX_MAX_RANKS || rank < 0 || rank >= nranks || nops < 0 ||
      slice_bytes < 4096 || slice_bytes % 4096 || !kinds || !counts || !dtypes)
    return fail(FMX_ERR_INVALID_ARG, "bad trace arguments");
  fmx_comm c;  // geometry only: no segment, no CUDA
  c.rank = rank;
  c.nranks = nranks;
  c.nslots = 2;
  if (const char* v = getenv("FMX_SLOTS")) c.nslots = std::min(FMX_MAX_SLOTS, std::max(2, atoi(v)));
  c.transport = transport == FMX_TRANSPORT_ZC ? FMX_TRANSPORT_ZC : FMX_TRANSPORT_CE;
  c.slice_bytes = slice_bytes;
  size_t max_bytes = 0;
  for (int i = 0; i < nops; ++i) max_bytes = std::max(max_bytes, counts[i] * (dtypes[i] ? 2 : 4));
  c.L = compute_layout(nranks, c.nslots, slice_bytes, max_bytes);
  c.total_bytes = c.L.total;
  if (const char* v = getenv("FMX_RESULT_VIA_CE")) c.result_via_ce = atoi(v) != 0;
  if (const char* v = getenv("FMX_GRAIN")) c.coarse = strcmp(v, "fine") != 0;
  c.coarse_gather = c.coarse;
  if (const char* v = getenv("FMX_GATHER_GRAIN")) c.coarse_gather = strcmp(v, "fine") != 0;
  if (const char* v = getenv("FMX_RAMP")) c.ramp = atoi(v) != 0;
  if (const char* v = getenv("FMX_LANES")) c.nlanes = std::min(3, std::max(1, atoi(v)));
  std::string out;
  TraceSink sink(&out);
  sink.nranks = nranks;
  // fake user buffers: only their offsets matter and they never reach SHM
  static char dummy[16] __attribute__((aligned(16)));
  for (int i = 0; i < nops; ++i) {
    int rc;
    sink.join();
    if (kinds[i] == 1 && (!roots || roots[i] < 0 || roots[i] >= nranks))
      return fail(FMX_ERR_INVALID_ARG, "bad broadcast root");
    if (kinds[i] == 0)
      rc = plan_allreduce(&c, sink, dummy, dummy, counts[i], dtypes[i], FMX_OP_SUM, 1.0f, true);
    else if (kinds[i] == 3 || kinds[i] == 4)  // reduce-scatter / all-gather, in place
      rc = plan_allreduce(&c, sink, dummy, dummy, counts[i], dtypes[i], FMX_OP_SUM, 1.0f, true,
                          kinds[i] == 3 ? kReduceScatter : kAllgather);
    else if (kinds[i] == 2)
      rc = plan_allreduce_host(&c, sink, 0, counts[i], dtypes[i], FMX_OP_SUM, 1.0f);
    else
      rc = plan_broadcast(&c, sink, dummy, dummy, counts[i], dtypes[i], roots ? roots[i] : 0);
    if (rc) return rc;
  }
  sink.join();
  if (used) *used = out.size() + 1;
  if (!buf || cap < out.size() + 1) return fail(FMX_ERR_INVALID_ARG, "trace buffer too small");
  memcpy(buf, out.c_str(), out.size() + 1);
  return FMX_OK;
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
  int rc = FMX_OK;
  const bool pushed = c->lane_ctx && g_ctx_push && g_ctx_push(c->lane_ctx) == CUDA_SUCCESS;
  if (c->has_done && cudaEventSynchronize(c->done) != cudaSuccess)
    rc = fail(FMX_ERR_CUDA, "pending collective failed: %s", cudaGetErrorString(cudaGetLastError()));
  if (c->done) cudaEventDestroy(c->done);
  if (c->fork) cudaEventDestroy(c->fork);
  for (int i = 0; i < kNumEvents; ++i)
    if (c->ev[i]) cudaEventDestroy(c->ev[i]);
  for (auto& pr : c->timed) {
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
  for (int l = 0; l < 2; ++l) {
    if (c->lane[l]) cudaStreamDestroy(c->lane[l]);
    if (c->joined[l]) cudaEventDestroy(c->joined[l]);
  }
  if (pushed) {
    CUcontext dummy;
    g_ctx_pop(&dummy);
  }
  if (c->scratch) cudaFree(c->scratch);
  if (c->stamps) cudaFree(c->stamps);
  if (c->registered) cudaHostUnregister(c->base);
  if (c->hdr) c->hdr->departed.fetch_add(1);
  unmap(c);
  delete c;
  return rc;
}

int fmx_comm_abort(fmx_comm_t c) {
  if (!c || !c->hdr) return fail(FMX_ERR_INVALID_ARG, "invalid communicator");
  c->hdr->aborted.store(1, std::memory_order_release);
  // Release every pending stream wait on every rank: push all counters far
  // ahead (cyclic >= compares, so +2^29 satisfies any outstanding target).
  for (int r = 0; r < c->nranks; ++r)
    for (int f = 0; f < kFlagsPerRank; ++f) {
      volatile uint32_t* p = c->flag_host(r, f);
      *p = *p + (1u << 29);
    }
  __sync_synchronize();
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

int fmx_comm_kernel_launches(fmx_comm_t c, uint64_t* launches) {
  if (!c || !launches) return fail(FMX_ERR_INVALID_ARG, "null argument");
  *launches = c->launches;
  return FMX_OK;
}

}  // extern "C"

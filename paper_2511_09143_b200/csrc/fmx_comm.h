// The communicator object and the schedule interface of libflexshm, shared by
// the CUDA half (flexshm_comm.cu: CudaSink, the C API) and the CUDA-free
// schedule (flexshm_plan.cpp: the plans, TraceSink, fmx_trace_plan).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstring>
#include <utility>
#include <vector>

#include "fmx_args.h"
#include "fmx_internal.h"

namespace fmx {
constexpr int kNumEvents = 2 * FMX_MAX_SLOTS + 12;  // W[K], G[K]; host path F[2], C[2],
                                                    // inputs, P[2]; reduce done (stage after
                                                    // reduce); fetch lane F[2], S[2]

// Round counters a flag's values follow (fmx_graph_*: baked flag values of a
// captured graph are re-based per replay by their counter's advance).
enum Counter { kCtrAr = 0, kCtrOs = 1, kCtrBc = 2, kCtrFence = 3, kNumCounters = 4 };

struct PendingGather;  // an allreduce's deferred last gather (flexshm_plan.cpp)

// The fused SGD epilogue of the allreduce being planned (fmx_allreduce_sgd):
// the owner's reduction updates its parameter piece and momentum shard.
struct SgdEpi {
  char* mom;  // momentum shard of this rank's owner chunk (null: momentum 0)
  float lr, mu, damp, wd;
  int nesterov, init;
};

// One batch-memop node of a captured graph that signals / waits on this
// communicator's flags, with its parameters as captured.
struct GraphMemop {
  CUgraphNode node;
  CUcontext ctx;
  unsigned int flags;
  std::vector<CUstreamBatchMemOpParams> ops;
  std::vector<int8_t> ctr;  // Counter of each op's flag (-1: not this communicator's)
};

// A captured graph (fmx_graph_capture_end): flag values as captured against
// counters c0, the counters' advance per replay, and the values last written
// into an instantiated graph.
struct GraphRec {
  uint32_t c0[kNumCounters] = {}, delta[kNumCounters] = {};
  uint64_t launches = 0;  // kernels per replay
  std::vector<GraphMemop> memops;
  CUgraphExec exec = nullptr;  // exec the `applied` offsets were written into
  uint32_t applied[kNumCounters] = {};
  bool live = true;
};
}  // namespace fmx

using fmx::Header;
using fmx::Layout;
using fmx::Stamp;

struct fmx_comm {
  int rank = -1, nranks = 0, nslots = 2, transport = FMX_TRANSPORT_CE, mig_aware = 1;
  size_t slice_bytes = 0, total_bytes = 0;
  Layout L{};
  char* base = nullptr;   // host VA of the mapping
  char* dbase = nullptr;  // device VA of the same bytes
  Header* hdr = nullptr;
  bool registered = false;
  uint32_t ar_round = 0, bc_round = 0, os_round = 0;
  int64_t barrier_gen = 0;
  char* scratch = nullptr;  // CE transport: n * slice_bytes of HBM
  cudaStream_t lane[3] = {};       // extra streams of lane 0 (stage, D2H) and lane 2 (gather, H2D); [1] unused
  cudaStream_t user = nullptr;      // caller's stream of the current collective (its input is ready there)
  cudaStream_t join_stream = nullptr;  // fmx_comm_set_join_stream: lane 1 runs here, not on `user`
  cudaStream_t completion = nullptr;   // stream the last collective completed on
  cudaStream_t last_main = nullptr;    // lane-1 stream of the last collective
  bool spin_wait = false;              // one-shot: OS_READY wait fused into the reduce kernel
                                       //   (MPS-concurrent ranks only; FMX_SPIN_WAIT=0/1 overrides)
  int reduce_ctas = 1184;              // grid cap of the reduce kernel (FMX_REDUCE_CTAS; local knob)
  int copy_ctas = 1184;                // CTA cap of one copy-kernel launch over all its segments
                                       // (FMX_COPY_CTAS; local knob: paces SM-side host stores)
  bool copy_fence = true;              // no-op kernel after every copy-engine batch (CudaSink::copy)
  bool fuse_signal = true;             // FMX_FUSE_SIGNAL=0: zero-copy stage + STAGED as two ops
  bool serialize = false;              // drain this rank's lanes before every kernel launch
                                       //   (under a kernel profiler / FMX_SERIALIZE=1)
  unsigned int* ctas_done = nullptr;   // device counters of the fused signal: [0] lane 0's
                                       //   stage copies, [1] the one-shot publish (lane 1)
  int last_class = -1;              // 0 device-buffer collective, 1 host path / broadcast
  CUcontext lane_ctx = nullptr;                // context the lane objects were created in
  cudaEvent_t ev[fmx::kNumEvents] = {};  // intra-rank lane sync (see the kEv* ids)
  cudaEvent_t fork = nullptr, joined[3] = {};
  bool result_via_ce = false;  // CE transport: result slot by copy engine, not SM stores
  bool copy2d = true;          // coalesce regular copy runs into cudaMemcpy2DAsync
  bool coarse = true;          // FMX_GRAIN=fine: per-piece waits instead of all-peer
  bool fine_first = false;     // FMX_GRAIN=first: per-contributor flags in round 0 only
  bool coarse_gather = true;   // FMX_GATHER_GRAIN=fine: per-owner gather waits only
  int ramp = 4;                // round geometry (allreduce_geometry): 4 remainder-sized first
                               // round (default); 0 equal rounds; 1/2/3 geometric ramps (slower)
  int min_rounds = 1;          // FMX_MIN_ROUNDS: shrink the slice so a chunk spans >= this many
  size_t zc_max = 2u << 20;    // FMX_ZC_MAX: AUTO transport moves messages <= this with SM copies

  // transport of one collective of `bytes`: AUTO picks zero-copy SM transfers
  // for small messages (no copy-engine launch latency: 0.12 vs 0.24 ms for
  // 1 KiB at 7 ranks) and the copy engines above zc_max (crossover 1-4 MiB, r01/r3j)
  bool use_zc(size_t bytes) const {
    return transport == FMX_TRANSPORT_ZC || (transport == FMX_TRANSPORT_AUTO && bytes <= zc_max);
  }
  // One-shot small-message allreduce (plan_allreduce_oneshot): every rank
  // publishes its whole buffer, one flag hop, every rank reduces all n in rank
  // order.  Taken by AUTO / ZC for messages up to oneshot_max bytes.
  size_t oneshot_max = 64u << 10;
  bool use_oneshot(size_t bytes) const {
    return transport != FMX_TRANSPORT_CE && transport != FMX_TRANSPORT_HOST && nranks > 1 &&
           bytes <= oneshot_max && bytes <= L.os_bytes;
  }
  // fmx_comm_set_defer: an allreduce's LAST gather is enqueued by the next
  // collective, after that one's first stage (or by fmx_comm_flush), so a
  // single in-order stream stages bucket b+1 while peers finish reducing b
  bool defer_gather = false;
  fmx::PendingGather* pending = nullptr;
  const fmx::SgdEpi* sgd = nullptr;  // set for the duration of one fmx_allreduce_sgd
  // FMX_STAGE_AFTER_REDUCE=1 (local knob: an intra-rank order only): stage(R+1)
  // waits for this rank's reduce(R), so the reduction's result store does not
  // share the D2H direction with this rank's next stage
  bool stage_after_reduce = false;
  bool stage_zc = false;       // FMX_STAGE_ZC=1 (local knob): stage by the SM copy kernel on CE
  bool fetch_lane = false;     // FMX_FETCH_LANE=1 (local knob): fetch on the gather lane into a
                               // double-buffered scratch (plan_allreduce)
  int rce_rounds = 8;          // with the fetch lane: result slot by copy engine from this many
                               // rounds (FMX_RCE_ROUNDS, local knob)
  int nlanes = 3;              // FMX_LANES=1: one stream; 2: gather on the reduce lane
  int join_lanes = 1;          // join-stream mode: 1 every lane on the join stream; 2 stage on
                               // its own stream; 3 stage and gather on their own (FMX_JOIN_LANES,
                               // local knob: stream mapping only, the schedule is the same)
  // live kernel timing (fmx_comm_set_timing): event pairs around every reduce
  bool timing = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> timed;
  size_t timed_used = 0;
  cudaEvent_t done = nullptr;
  bool has_done = false;
  uint64_t launches = 0;
  // pipeline timeline probe (fmx_comm_set_stamps): device ring of Stamp entries
  fmx::Stamp* stamps = nullptr;
  size_t stamp_cap = 0, stamp_used = 0;
  std::vector<fmx_peer_info> peers;
  std::vector<uint32_t> abort_target;  // fmx_comm_abort: raised flag values (re-asserted)
  std::vector<CUstreamBatchMemOpParams> ops;

  // CUDA-graph capture (fmx_graph_*).  While a capture is active (cap_active =
  // its id) every collective is recorded into the caller's stream capture with
  // flag values from the counters; events remember the capture they were last
  // recorded in (0: eager) and a wait on an event of another capture / of the
  // eager timeline is dropped: that ordering comes from the stream order of
  // graph launches and the fence every replay ends with.
  uint32_t fence_round = 0;
  int cap_active = 0, cap_next = 0;
  uint32_t cap_c0[fmx::kNumCounters] = {};
  uint64_t cap_launches0 = 0;
  int ev_cap[fmx::kNumEvents] = {};
  int done_cap = 0;
  bool fenced = true;                    // no collective since the last fence / replay
  bool cap_fenced = true;                // `fenced` when the capture began (nothing captured runs)
  cudaStream_t graph_stream = nullptr;   // stream of the last replay (ordering of the next call)
  cudaEvent_t graph_ev = nullptr;
  std::vector<fmx::GraphRec> graphs;
  uint32_t* counter(int k) {
    return k == fmx::kCtrAr ? &ar_round : k == fmx::kCtrOs ? &os_round
                                        : k == fmx::kCtrBc ? &bc_round : &fence_round;
  }

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
  size_t os_slot_off(uint32_t J, int r) const {
    return L.os_off + ((size_t)(J % fmx::kOsSlots) * nranks + r) * L.os_bytes;
  }
  size_t user_region_off(int r) const { return L.user_off + (size_t)r * L.user_bytes; }
  // host (dev=false) or device (dev=true) address of a segment offset
  char* at(bool dev, size_t off) const { return (dev ? dbase : base) + off; }
  CUdeviceptr flag_dev(int r, int f) const {
    return (CUdeviceptr)(dbase + L.flags_off + ((size_t)r * fmx::kFlagsPerRank + f) * 64);
  }
  volatile uint32_t* flag_host(int r, int f) const {
    return (volatile uint32_t*)(base + L.flags_off + ((size_t)r * fmx::kFlagsPerRank + f) * 64);
  }
};


namespace fmx {

inline cudaStream_t lane_stream(const fmx_comm* c, int lane) {
  // lane 1 runs on the main stream: the join stream if one is set, else the
  // caller's.  Only lanes 0 and 2 are extra streams: with 7 MPS clients per
  // GPU, a third extra stream per client made the allreduce 1.5x slower
  // (streams alias onto shared hardware queues; profiles/r01/r2q).
  cudaStream_t main = c->join_stream ? c->join_stream : c->user;
  // join-stream mode runs every lane on the join stream: next to the caller's
  // compute stream, two more extra streams per MPS client made bucketed
  // allreduces 2.5x slower (hardware-queue aliasing, profiles/r01/r2w), and a
  // single in-order stream per rank is as fast as three lanes on this box
  if (c->nlanes == 1 || lane == 1) return main;
  if (c->join_stream) {
    const int jl = std::min(c->join_lanes, c->nlanes);
    if (jl <= 1 || (lane == 2 && jl < 3)) return main;
    return c->lane[lane];
  }
  if (c->nlanes == 2) return lane == 0 ? c->lane[0] : main;
  return c->lane[lane];
}


// ---- the plan: what one rank enqueues for one collective -----------------------
//
// plan_allreduce / plan_broadcast describe the schedule once, against a Sink.
// Work is issued on three lanes per rank so the link directions overlap inside
// a rank: lane 0 stages (HBM -> SHM, D2H), lane 1 fetches and reduces
// (SHM -> HBM, H2D; the caller's or the join stream), lane 2 gathers (H2D).
// Lanes fork from / join back into the main stream at every collective
// (on_lanes, flexshm_comm.cu).  CudaSink turns the
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
  // wait until every peer's `flag` >= v, then reduce (a sink may fuse the two)
  virtual int wait_reduce(int lane, const PlanReduce& r, int flag, uint32_t v, int skip) {
    int rc = wait_peers(lane, flag, v, skip);
    return rc ? rc : reduce(lane, r);
  }
  virtual int signal(int lane, int flag, uint32_t v) = 0;
  // copy, then signal `flag` = v on the same lane (a sink may fuse the two)
  virtual int copy_signal(int lane, const std::vector<PlanSeg>& segs, bool src_sys,
                          bool use_kernel, int flag, uint32_t v) {
    int rc = copy(lane, segs, src_sys, use_kernel);
    return rc ? rc : signal(lane, flag, v);
  }
  virtual int signal2(int lane, int f0, uint32_t v0, int f1, uint32_t v1) = 0;
  virtual int wait_peers(int lane, int flag, uint32_t v, int skip) = 0;
  virtual int wait_rank(int lane, int q, int flag, uint32_t v) = 0;
  virtual int d2d(int lane, void* dst, const void* src, size_t bytes, Annot from, Annot to) = 0;
  // intra-rank lane ordering through CUDA events (enqueue-order semantics)
  virtual int record(int lane, int ev) = 0;
  virtual int wait_event(int lane, int ev) = 0;
  // host-program accesses to SHM around a collective (trace only)
  virtual int host_access(int lane, const Annot& a, bool write) { return FMX_OK; }
  // user-buffer scope of the collective being planned (TraceSink: each
  // collective's buffer is a separate range); a deferred gather keeps its own
  virtual int64_t scope() const { return 0; }
  virtual void set_scope(int64_t) {}
};


// Round geometry of one collective (allreduce_geometry, flexshm_plan.cpp).
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
Geometry allreduce_geometry(const fmx_comm* c, size_t count, int dtype, size_t chunk_elems = 0);

inline Annot ubuf(size_t off_bytes, size_t bytes) { return Annot{(int64_t)off_bytes, bytes, -1, 0}; }
inline Annot sbuf(size_t off_bytes, size_t bytes) { return Annot{(int64_t)off_bytes, bytes, -1, 0, true}; }


// The three owner-chunk collectives of plan_allreduce.
enum Kind { kAllreduce = 0, kReduceScatter = 1, kAllgather = 2 };

// The schedule settings (Proto) from this process's environment, and their
// application to a communicator (rank 0 publishes, every rank applies).
Proto proto_from_env();
void apply_proto(fmx_comm* c, const Proto& p);

int plan_allreduce(fmx_comm* c, Sink& k, const char* src, char* dst, size_t count, int dtype,
                   int op, float factor, bool aligned, int kind = kAllreduce);
int plan_allreduce_oneshot(fmx_comm* c, Sink& k, const char* src, char* dst, size_t count,
                           int dtype, int op, float factor, bool aligned);
int plan_allreduce_host(fmx_comm* c, Sink& k, size_t off_bytes, size_t count, int dtype, int op,
                        float factor);
int plan_broadcast(fmx_comm* c, Sink& k, const char* src, char* dst, size_t count, int dtype,
                   int root);
// enqueue the pending deferred gather, if any (every plan does this first)
int plan_flush(fmx_comm* c, Sink& k);
// fmx_comm_fence: flush, signal FENCE, wait for every peer's FENCE (lane 1)
int plan_fence(fmx_comm* c, Sink& k);
void drop_pending(fmx_comm* c);

}  // namespace fmx

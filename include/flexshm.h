/*
 * flexshm.h - C ABI of libflexshm.so, the B200-native one-to-many data path
 * of Flex-MIG (arxiv 2511.09143): a data-parallel job spread over many 1g
 * instances (MIG slices, or SM-partitioned stand-ins) joined by a
 * host-shared-memory allreduce / broadcast.
 *
 * Plain C types only (no torch / CUDA types in the signatures): device
 * buffers are `void*` device pointers, the stream is a `void*` that holds a
 * cudaStream_t.  Every call returns an int status, 0 = FMX_OK.
 *
 * What each entry point replaces (reference file:line, /root/reference):
 *
 *   fmx_validate_peers  <- migsim.commsim.discover_peers
 *                          (pkg/src/migsim/commsim.py:67-88) and
 *                          PeerInfo.__post_init__ (commsim.py:35-42)
 *   fmx_topology        <- migsim.commsim.build_topology (commsim.py:91-116)
 *   fmx_restore_bus_id  <- migsim.commsim.restore_bus_id (commsim.py:119-123)
 *   fmx_comm_init       <- the paper's patched ncclCommInitRank: bootstrap
 *                          allgather of peer info incl. mig_id, duplicate
 *                          check, synthetic bus-id labels;
 *                          shaped like ncclCommInitRank (nccl.h:160)
 *   fmx_allreduce       <- ncclAllReduce over the SHM transport, reached from
 *                          DDP (nccl.h:379)
 *   fmx_broadcast       <- ncclBroadcast (ZeRO shard / DDP init broadcast,
 *                          PAPER.md:485; nccl.h:392)
 *   fmx_reduce_scatter  <- ncclReduceScatter (nccl.h:408)
 *   fmx_allgather       <- ncclAllGather (inference jobs, PAPER.md:485;
 *                          nccl.h:425)
 *   fmx_comm_destroy / fmx_comm_abort <- ncclCommDestroy / ncclCommAbort
 *   fmx_comm_fence, fmx_comm_set_defer / fmx_comm_flush, fmx_graph_*
 *                       <- no reference interface: what makes the collectives
 *                          usable inside a CUDA-graph-captured DP step (NCCL's
 *                          analog is capturing ncclAllReduce under
 *                          cudaStreamBeginCapture); DESIGN.md §3.3-3.4
 *
 * Status codes map 1:1 to Python exceptions (paper_2511_09143_b200/_lib.py):
 * DUPLICATE_DEVICE -> DuplicateDeviceError(rank_a, rank_b) with the same
 * (earlier, later) pair as commsim.py:85-86; MALFORMED_LABEL ->
 * MalformedLabelError; BAD_RANKS / EMPTY_MIG_ID / INVALID_ARG -> ValueError.
 *
 * Threading: one communicator per rank process (several per process are
 * allowed for in-process testing); calls on one communicator must be
 * serialised by the caller (the NCCL rule).  Collectives are asynchronous on
 * the given stream; init and destroy are blocking.
 */
#ifndef FLEXSHM_H
#define FLEXSHM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FMX_ABI_VERSION 1
#define FMX_BUS_ID_LEN 16   /* "XX:XX:XX.0" + NUL, padded */
#define FMX_MIG_ID_LEN 128
#define FMX_MAX_RANKS 64
#define FMX_MAX_RANKS_PER_BUS 10
#define FMX_MAX_SLOTS 4 /* pipeline depth limit (slots per SHM region) */

enum fmx_status {
  FMX_OK = 0,
  FMX_ERR_DUPLICATE_DEVICE = 1, /* two ranks bound to one device (commsim.py:85-86) */
  FMX_ERR_MALFORMED_LABEL = 2,  /* non-canonical bus id, or > 10 ranks per bus */
  FMX_ERR_BAD_RANKS = 3,        /* ranks not exactly 0..n-1 (commsim.py:76-77) */
  FMX_ERR_EMPTY_MIG_ID = 4,     /* PeerInfo with empty mig_id (commsim.py:41-42) */
  FMX_ERR_INVALID_ARG = 5,
  FMX_ERR_CUDA = 6,
  FMX_ERR_SHM = 7,
  FMX_ERR_TIMEOUT = 8,
  FMX_ERR_ABORTED = 9,
  FMX_ERR_UNSUPPORTED = 10
};

enum fmx_dtype { FMX_FLOAT32 = 0, FMX_BFLOAT16 = 1 };

/* Scale conventions; the arithmetic is the fixed ascending-rank fp32 sum.
 *
 * DDP's mean is FMX_OP_PREMUL_SUM with factor = fl32(1/world): the default
 * hook's `bucket.div_(world)` (torch/distributed/algorithms/ddp_comm_hooks/
 * default_hooks.py:26) runs ATen's div_true_kernel_cuda, which for a CPU
 * scalar divisor computes a * fl32(1/b) in fp32 (BinaryDivTrueKernel.cu),
 * and the hook-less reducer multiplies by 1/div_factor; NCCL's equivalent is
 * ncclRedOpCreatePreMulSum (nccl.h:314).  For bf16 each product is rounded
 * to bf16 (the bucket is a bf16 tensor after the in-place scale).
 * FMX_OP_PREDIV_SUM keeps IEEE true division as an explicit op. */
enum fmx_op {
  FMX_OP_SUM = 0,           /* out = x0 + x1 + ... (left to right)            */
  FMX_OP_SUM_POSTSCALE = 1, /* out = (sum) * factor                           */
  FMX_OP_PREDIV_SUM = 2,    /* out = x0/factor + x1/factor + ... (true divide) */
  FMX_OP_PREMUL_SUM = 3     /* out = x0*factor + x1*factor + ... (DDP mean     */
                            /* with factor = fl32(1/world); ncclPreMulSum)     */
};

/* How host-link bytes move.  ZC: SM kernels store to / load from the mapped
 * SHM segment (128-bit, zero-copy).  CE: copy engines move the bytes, SM
 * kernels reduce out of HBM.  AUTO picks per collective by size: ZC up to
 * 2 MiB (no copy-engine launch latency), CE above (faster at bandwidth across
 * processes on one GPU; env FMX_ZC_MAX overrides the cut).  HOST joins the bootstrap and host barrier without
 * touching CUDA (collectives then return FMX_ERR_UNSUPPORTED); it is how the
 * multi-process bootstrap is exercised on GPU-less machines. */
enum fmx_transport {
  FMX_TRANSPORT_AUTO = 0,
  FMX_TRANSPORT_ZC = 1,
  FMX_TRANSPORT_CE = 2,
  FMX_TRANSPORT_HOST = 3 /* bootstrap + barrier only, no CUDA calls at all */
};

/* One rank's identity (commsim.PeerInfo, commsim.py:27-42). */
typedef struct fmx_peer_info {
  int32_t rank;
  char pcie_bus_id[FMX_BUS_ID_LEN]; /* canonical "XX:XX:XX.0" (upper case)   */
  char mig_id[FMX_MIG_ID_LEN];      /* MIG UUID or "GC-<gpu uuid>-<slot>"   */
  int64_t host_hash;
  int64_t pid_hash;
} fmx_peer_info;

typedef struct fmx_comm* fmx_comm_t;

/* ---- host-only bootstrap rules (no GPU needed) ---------------------------- */

/* Normalise + validate one PeerInfo in place (upper-cases the bus id). */
int fmx_check_peer(fmx_peer_info* peer);

/* discover_peers: ranks must be 0..n-1; duplicate key (host, bus, mig_id),
 * or (host, bus) when mig_aware == 0.  On FMX_ERR_DUPLICATE_DEVICE,
 * *rank_a / *rank_b receive the (earlier, later) pair. */
int fmx_validate_peers(const fmx_peer_info* peers, int n, int mig_aware,
                       int* rank_a, int* rank_b);

/* build_topology over peers in rank order: labels[i] (FMX_BUS_ID_LEN chars)
 * is rank i's label; mig_buses / mig_counts (n entries) receive the mig_list
 * in first-seen order, *n_buses its length. */
int fmx_topology(const fmx_peer_info* peers, int n, char* labels, char* mig_buses,
                 int* mig_counts, int* n_buses);

/* restore_bus_id: "00:4B:00.3" -> "00:4B:00.0"; out has FMX_BUS_ID_LEN bytes. */
int fmx_restore_bus_id(const char* label, char* out);

/* ---- communicator ---------------------------------------------------------- */

/* Collective over all `nranks` processes calling it with the same job_key.
 * Rank 0 creates POSIX SHM "/fmx-<job_key>", every rank publishes `self`,
 * the table is validated with the rules above (mig_aware), the segment is
 * pinned and device-mapped (cudaHostRegister Mapped|Portable) in the calling
 * thread's current CUDA context.  slice_bytes = bytes per (owner,
 * contributor) pipeline slot, 0 = default (4 MiB; 16 MiB at two ranks);
 * nslots = pipeline depth, 2 (double buffering) .. FMX_MAX_SLOTS, 0 = default
 * (2; 4 at two ranks; env FMX_SLOTS overrides).  host_bytes =
 * size of every rank's registered host buffer (fmx_host_buffer), 0 = none.
 * Rank 0's slice_bytes / nslots / host_bytes win, and so do the schedule
 * settings of rank 0's environment (FMX_RAMP, FMX_MIN_ROUNDS, FMX_GRAIN,
 * FMX_GATHER_GRAIN, FMX_LANES, FMX_RESULT_VIA_CE, FMX_ZC_MAX, FMX_ONESHOT_MAX), published in
 * the segment header so every rank runs the same protocol.  Peers on another
 * host (different host_hash: the reference's select_transport answers "NET",
 * commsim.py:126-132) are refused with FMX_ERR_UNSUPPORTED: the transport is
 * one host's shared memory.  timeout_s bounds every bootstrap wait. */
int fmx_comm_init(fmx_comm_t* comm, const char* job_key, int nranks, int rank,
                  const fmx_peer_info* self, int mig_aware, size_t slice_bytes, int nslots,
                  size_t host_bytes, int transport, double timeout_s);

/* In-place allowed (send == recv).  count elements of dtype; op/factor per
 * enum fmx_op.  Enqueued on `stream` (a cudaStream_t); returns immediately.
 * Messages up to FMX_ONESHOT_MAX bytes (64 KiB; AUTO / ZC transports) take the
 * one-shot path: every rank publishes its buffer, one flag hop, every rank
 * reduces all n contributions in rank order - same bits as the pipelined
 * reduce-scatter / all-gather used above that size. */
int fmx_allreduce(fmx_comm_t comm, const void* send, void* recv, size_t count, int dtype,
                  int op, float factor, void* stream);

/* Fused optimizer step (fp32): allreduce of `grad` (op SUM or PREMUL_SUM, as
 * fmx_allreduce) in which each OWNER applies torch's SGD step (torch/optim/
 * sgd.py _multi_tensor_sgd: weight decay, momentum with dampening, Nesterov)
 * to its chunk of `param` with the reduced gradient, and the all-gather then
 * distributes the updated parameters into every rank's `param` - the
 * optimizer fused into the collective's reduction, each element stepped once
 * instead of on every rank (ZeRO-1 style: `momentum` holds only this rank's
 * shard, fmx_allreduce_shard's len elements, fp32, 16-byte aligned).  `grad`
 * is left as it was.  Bit-identical to every rank running torch's SGD on the
 * averaged gradient (tests/test_graph_dp_gpu.py). */
typedef struct fmx_sgd {
  float lr, momentum, dampening, weight_decay;
  int nesterov;
  int first_step; /* 1: the momentum shard is initialised to the gradient (torch's first step) */
} fmx_sgd;
int fmx_allreduce_sgd(fmx_comm_t comm, const void* grad, void* param, void* momentum, size_t count,
                      int op, float factor, const fmx_sgd* sgd, void* stream);
/* This rank's owner chunk of an allreduce of `count` elements: [*offset, *offset + *len). */
int fmx_allreduce_shard(fmx_comm_t comm, size_t count, int dtype, size_t* offset, size_t* len);

/* Root's send buffer -> every rank's recv buffer (bit copy). */
int fmx_broadcast(fmx_comm_t comm, const void* send, void* recv, size_t count, int dtype,
                  int root, void* stream);

/* NCCL layout: send holds nranks*recvcount elements, rank r receives the
 * rank-order reduction (op/factor as fmx_allreduce) of elements
 * [r*recvcount, (r+1)*recvcount) in recv.  In place when
 * recv == send + rank*recvcount. */
int fmx_reduce_scatter(fmx_comm_t comm, const void* send, void* recv, size_t recvcount, int dtype,
                       int op, float factor, void* stream);

/* NCCL layout: every rank's sendcount elements land at recv[r*sendcount] of
 * every rank (bit copy).  In place when send == recv + rank*sendcount. */
int fmx_allgather(fmx_comm_t comm, const void* send, void* recv, size_t sendcount, int dtype,
                  void* stream);

/* Registered host buffers (the NCCL user-buffer-registration idea for host
 * memory): every rank owns a pinned, device-mapped region of host_bytes inside
 * the segment; any rank's region can be mapped (for inspection).  */
int fmx_host_buffer(fmx_comm_t comm, int rank, void** ptr, size_t* bytes);

/* Allreduce of host-resident data, in place over every rank's region bytes
 * [offset, offset + count*size(dtype)): the GPU reads each owner's chunk out of
 * all regions and writes the rank-order result back into all regions - no
 * staging copy and no all-gather (k*S H2D + k*S D2H per GPU).  Same
 * arithmetic and op/factor semantics as fmx_allreduce.  The caller must have
 * finished writing its region before the call and may read it after the
 * stream has drained. */
int fmx_allreduce_host(fmx_comm_t comm, size_t offset, size_t count, int dtype, int op,
                       float factor, void* stream);

/* The owner-side reduction kernel on its own (no communicator): dst[i] =
 * rank-order fp32 sum of srcs[0..nsrc)[i] with the op/factor convention,
 * optionally also stored to dst_sys (mapped host memory, zero-copy).  Bit
 * `q` of sys_mask marks srcs[q] as mapped host memory (cache-volatile loads).
 * Used to test the kernel against the oracle and to time it in isolation. */
int fmx_reduce_local(const void* const* srcs, int nsrc, uint64_t sys_mask, void* dst,
                     void* dst_sys, size_t count, int dtype, int op, float factor, void* stream);

/* Host-side barrier over the communicator (SHM counter; no GPU work). */
int fmx_barrier(fmx_comm_t comm, double timeout_s);

int fmx_comm_destroy(fmx_comm_t comm);
/* Marks the communicator aborted and releases every stream wait of every
 * rank on it (results of in-flight collectives are undefined). */
int fmx_comm_abort(fmx_comm_t comm);

int fmx_comm_rank(fmx_comm_t comm, int* rank);
int fmx_comm_count(fmx_comm_t comm, int* nranks);
int fmx_comm_peer(fmx_comm_t comm, int rank, fmx_peer_info* out);
/* Effective configuration: slice bytes, transport, segment bytes. */
int fmx_comm_config(fmx_comm_t comm, size_t* slice_bytes, int* transport, size_t* shm_bytes);
/* Snapshot of every rank's flag counters (nranks x 4: STAGED, REDUCED,
 * BC_STAGED, BC_DONE), read from host memory - for hang diagnosis. */
int fmx_comm_flags(fmx_comm_t comm, uint32_t* out, int cap);
/* Timeline probe: poll every flag of every rank (host reads of the segment,
 * no GPU involvement) for `seconds` and record each change as two uint64s:
 * ns since the call, and (rank << 48 | flag << 32 | value).  *n_out = number
 * of changes.  Flag ids: 0 STAGED, 1 REDUCED, 2 BC_STAGED, 3 BC_DONE,
 * 8 + o STAGED_TO[o]. */
int fmx_comm_monitor(fmx_comm_t comm, double seconds, uint64_t* out, size_t cap, size_t* n_out);

/* Completion stream.  By default a collective forks from the stream it is
 * called on and joins back into it.  With a join stream set (non-null), it
 * still forks from the call's stream (its input is ready there) but runs ALL
 * of its lanes, in order, on `stream` and completes there: the calling stream
 * (e.g. DDP's autograd stream) runs on and never waits for a collective.
 * Consecutive collectives are ordered on the join stream; they do not overlap
 * inside the library (extra lane streams next to a compute stream aliased
 * hardware queues under MPS and were slower).  The caller
 * orders reuse of a buffer after its completion (as DDP does by waiting on the
 * bucket future).  NULL restores the default. */
int fmx_comm_set_join_stream(fmx_comm_t comm, void* stream);
/* The stream the last collective completed on: the calling stream by
 * default, the join stream in join-stream mode.  Make consumers wait for an
 * event recorded on it. */
int fmx_comm_completion_stream(fmx_comm_t comm, void** stream);

/* Live timing of the reduction kernel: with timing on, every reduce launch
 * is bracketed by CUDA events on the lane stream it runs on; kernel_time
 * returns the summed device time and the number of timed launches since
 * timing was (re)enabled.  Used by bench.py for the per-kernel roofline. */
int fmx_comm_set_timing(fmx_comm_t comm, int on);
int fmx_comm_kernel_time(fmx_comm_t comm, double* total_ms, uint64_t* count);
/* Pipeline timeline probe.  set_stamps(capacity > 0) allocates a device ring
 * of `capacity` entries and, from then on, enqueues after every operation
 * (copy batch, reduction, flag signal, flag / event wait) a one-thread kernel
 * that records the GPU global timer (one clock for all processes on a GPU)
 * with a (lane << 8 | op) tag and an info word; capacity 0 turns it off.
 * fmx_comm_stamps synchronises the device and returns up to cap/2 entries as
 * pairs (t_ns, tag << 32 | info).  Op kinds: 1 wait-peers, 2 wait-rank,
 * 3 wait-event, 4 copy (info = bytes), 5 reduce (info = elements), 6 signal
 * (info = value).  Stamp kernels are not counted by fmx_comm_kernel_launches. */
int fmx_comm_set_stamps(fmx_comm_t comm, size_t capacity);
int fmx_comm_stamps(fmx_comm_t comm, uint64_t* out, size_t cap, size_t* n_out);
/* A caller's marker on the same timeline (op kind 7, lane 15): e.g. the start
 * and end of a training step on the compute stream. */
int fmx_comm_stamp(fmx_comm_t comm, void* stream, uint32_t info);
/* Number of device kernels this communicator has launched so far. */
int fmx_comm_kernel_launches(fmx_comm_t comm, uint64_t* launches);

/* ---- fences and CUDA graphs ------------------------------------------------ */

/* Fence: enqueued on `stream` after every earlier collective of this rank; it
 * completes once every rank reached its own fence (signal FENCE, wait for
 * every peer's).  After it, no peer touches any SHM slot of an earlier
 * collective. */
int fmx_comm_fence(fmx_comm_t comm, void* stream);

/* Deferred gather (set_defer on): an allreduce's last all-gather round is
 * enqueued by this rank's NEXT collective, right after that one's first stage,
 * or by fmx_comm_flush - so on one in-order stream (join-stream mode) the
 * stage of bucket b+1 fills the wait for peers to finish reducing bucket b.
 * An allreduce's result is complete only after the next collective / flush
 * (on the stream that one runs on).  Off by default; turning it off needs no
 * pending gather. */
int fmx_comm_set_defer(fmx_comm_t comm, int on);
int fmx_comm_flush(fmx_comm_t comm, void* stream);

/* Capture collectives into a CUDA graph (a whole DP training step, replayed
 * as one launch: ddp.ShmDataParallel).  No reference interface: NCCL
 * collectives are capturable (ncclGroup under cudaStreamBeginCapture), and
 * this is how the SHM path is.
 *   capture_begin  before the caller begins the stream capture;
 *   capture_end    after it ended, with the captured cudaGraph_t, BEFORE it
 *                  is instantiated: appends the end-of-replay fence after every
 *                  leaf and records the graph's flag operations -> *handle
 *                  (graph NULL: abandon a failed capture);
 *   launch_prepare before EVERY launch of an instance (cudaGraphExec_t) of
 *                  that graph on `stream`, followed by exactly one launch:
 *                  re-bases the instance's flag values to the communicator's
 *                  round counters (and fences first if collectives ran since
 *                  the last replay).
 * Replays of one communicator's graphs and its eager calls are ordered by the
 * streams they are issued on (a replay on another stream than the previous
 * one waits for it).  Every rank must capture and replay the same sequence. */
int fmx_graph_capture_begin(fmx_comm_t comm);
int fmx_graph_capture_end(fmx_comm_t comm, void* graph, int* handle);
int fmx_graph_launch_prepare(fmx_comm_t comm, int handle, void* graph_exec, void* stream);
int fmx_graph_release(fmx_comm_t comm, int handle);

/* ---- schedule introspection (no GPU, no segment) ---------------------------- */

/* Write the schedule `rank` of an `nranks` communicator would enqueue for a
 * sequence of `nops` collectives (kinds[i]: 0 allreduce, 1 broadcast with
 * roots[i], 2 host-buffer allreduce, 3 reduce-scatter and 4 all-gather with
 * counts[i] per rank, 5 fmx_comm_flush) as text (environment: FMX_TRACE_OVERLAP
 * join-stream mode, FMX_TRACE_DEFER deferred gather, FMX_TRACE_REPLAYS=k the
 * sequence as a captured graph replayed k times): one line per SHM access ("W off bytes round", "R off
 * bytes writer round") or flag op ("S flag value", "A rank flag value"),
 * "#" between collectives.  Used to model-check the protocol for any world
 * size on a CPU (tests/test_protocol_model.py).  *used = bytes needed. */
int fmx_trace_plan(int nranks, int rank, int transport, size_t slice_bytes, int nops,
                   const int* kinds, const size_t* counts, const int* dtypes, const int* roots,
                   char* buf, size_t cap, size_t* used);

/* ---- diagnostics ----------------------------------------------------------- */

const char* fmx_last_error(void);           /* thread-local message          */
int fmx_dup_ranks(int* rank_a, int* rank_b); /* pair of the last DUPLICATE    */
int fmx_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* FLEXSHM_H */

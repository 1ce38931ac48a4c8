// The schedule of libflexshm: what one rank enqueues for one collective,
// written once against a Sink.  CudaSink (flexshm_comm.cu) turns it into
// stream operations; TraceSink (here) records it as text so every rank of any
// world size can be model-checked on a CPU (fmx_trace_plan,
// tests/test_protocol_model.py).  No CUDA calls in this file.
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "fmx_comm.h"

namespace fmx {

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
  int signal(int lane, int flag, uint32_t v) override {
    return line("%d S %d %u\n", lane, flag, v + off(flag));
  }
  int signal2(int lane, int f0, uint32_t v0, int f1, uint32_t v1) override {
    line("%d S %d %u\n", lane, f0, v0 + off(f0));
    return line("%d S %d %u\n", lane, f1, v1 + off(f1));
  }
  int wait_peers(int lane, int flag, uint32_t v, int skip) override {
    for (int q = 0; q < nranks; ++q)
      if (q != skip) line("%d A %d %d %u\n", lane, q, flag, v + off(flag));
    return FMX_OK;
  }
  int wait_rank(int lane, int q, int flag, uint32_t v) override {
    return line("%d A %d %d %u\n", lane, q, flag, v + off(flag));
  }
  int d2d(int lane, void*, const void*, size_t, Annot from, Annot to) override {
    user(lane, from, false);
    user(lane, to, true);
    return FMX_OK;
  }
  int record(int lane, int ev) override {
    ev_epoch_[ev] = epoch;
    return line("%d E %d %d\n", lane, ev, ++seq_[ev]);
  }
  // (a replayed graph drops waits on events recorded outside its capture)
  int wait_event(int lane, int ev) override {
    return seq_[ev] && ev_epoch_[ev] == epoch ? line("%d X %d %d\n", lane, ev, seq_[ev]) : FMX_OK;
  }
  int host_access(int lane, const Annot& a, bool write) override {
    shm(lane, a, write);
    return FMX_OK;
  }
  int join() { return line("J\n"); }
  int64_t scope() const override { return user_base; }
  void set_scope(int64_t b) override { user_base = b; }
  int nranks = 0;
  int64_t user_base = 0;  // overlap traces: each collective's user buffer is a separate range
  // graph replays (FMX_TRACE_REPLAYS): flag values re-based per counter class
  // (what fmx_graph_launch_prepare writes into the nodes), annotation rounds
  // tagged with the replay, events of other replays invisible
  uint32_t flag_off[kNumCounters] = {};
  uint32_t round_tag = 0;
  int epoch = 0;

 private:
  void shm(int lane, const Annot& a, bool write) {
    if (a.off < 0 || a.bytes == 0) return;
    if (write)
      line("%d W %lld %zu %u\n", lane, (long long)a.off, a.bytes, a.round + round_tag);
    else
      line("%d R %lld %zu %d %u\n", lane, (long long)a.off, a.bytes, a.writer, a.round + round_tag);
  }
  void user(int lane, const Annot& a, bool write) {
    if (a.off < 0 || a.bytes == 0) return;
    const char* kind = a.scratch ? (write ? "SW" : "SR") : (write ? "UW" : "UR");
    line("%d %s %lld %zu\n", lane, kind, (long long)(a.off + (a.scratch ? 0 : user_base)), a.bytes);
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
  uint32_t off(int flag) const {
    const int k = (flag == kStaged || flag == kReduced || flag >= kStagedTo) ? kCtrAr
                  : flag == kOsReady                                      ? kCtrOs
                  : flag == kFence                                        ? kCtrFence
                                                                          : kCtrBc;
    return flag_off[k];
  }
  std::string* out_;
  int seq_[kNumEvents] = {};
  int ev_epoch_[kNumEvents] = {};
};

Proto proto_from_env() {
  Proto p{};
  p.ramp = 4;  // remainder-sized first round: 26.7 vs 27.4 ms for the ResNet-50 gradient (r02/r2d)
  p.min_rounds = 1;
  p.coarse = 1;
  p.fine_first = 0;
  p.nlanes = 3;
  p.result_via_ce = 0;
  p.zc_max = 2u << 20;
  p.oneshot_max = 64 << 10;
  if (const char* v = getenv("FMX_RESULT_VIA_CE")) p.result_via_ce = atoi(v) != 0;
  if (const char* v = getenv("FMX_GRAIN")) {
    p.coarse = strcmp(v, "fine") != 0;
    p.fine_first = strcmp(v, "first") == 0;
  }
  p.coarse_gather = p.coarse;
  if (const char* v = getenv("FMX_GATHER_GRAIN")) p.coarse_gather = strcmp(v, "fine") != 0;
  if (const char* v = getenv("FMX_LANES")) p.nlanes = std::min(3, std::max(1, atoi(v)));
  if (const char* v = getenv("FMX_RAMP")) p.ramp = atoi(v);
  if (const char* v = getenv("FMX_MIN_ROUNDS")) p.min_rounds = atoi(v);
  if (const char* v = getenv("FMX_ZC_MAX")) p.zc_max = strtoull(v, nullptr, 10);
  if (const char* v = getenv("FMX_ONESHOT_MAX"))
    p.oneshot_max = (int32_t)std::min<long long>(std::max(0ll, atoll(v)), (long long)kOneShotCap);
  return p;
}

void apply_proto(fmx_comm* c, const Proto& p) {
  c->ramp = p.ramp;
  c->min_rounds = p.min_rounds;
  c->coarse = p.coarse != 0;
  c->fine_first = p.fine_first != 0;
  c->coarse_gather = p.coarse_gather != 0;
  c->nlanes = p.nlanes;
  c->result_via_ce = p.result_via_ce != 0;
  c->zc_max = p.zc_max;
  c->oneshot_max = (size_t)std::max(0, p.oneshot_max);
}

// Round j of every chunk covers [prefix(j), prefix(j) + size(j)).  By default
// (FMX_RAMP=4) every round is one full slice except the first, which takes
// the remainder: the same number of rounds as an equal split, with a shorter
// pipeline fill (2.5 % faster on the ResNet-50 gradient, profiles/r02/r2d).
// FMX_RAMP=0 splits equally; FMX_RAMP=1 makes the first rounds slice/8, /4,
// /2 and the last ones /2, /4, /8, FMX_RAMP=2 ramps up only, FMX_RAMP=3 adds
// one quarter-slice first round; those measured slower (extra rounds cost
// more than the fill they save).
// chunk_elems = 0: allreduce chunking (16-byte aligned chunk starts over
// `count`); otherwise every rank's chunk has exactly chunk_elems elements and
// count = n * chunk_elems (reduce-scatter / all-gather, NCCL's layout).
Geometry allreduce_geometry(const fmx_comm* c, size_t count, int dtype, size_t chunk_elems) {
  Geometry g;
  const int n = c->nranks;
  g.esz = dtype == FMX_FLOAT32 ? 4 : 2;
  const size_t vec = 16 / g.esz;
  g.count = chunk_elems ? chunk_elems * n : count;
  g.chunk = chunk_elems ? chunk_elems : ((count + n - 1) / n + vec - 1) / vec * vec;
  g.slice = c->slice_bytes / g.esz;
  if (c->min_rounds > 1) {
    // small collectives (a DDP bucket is one chunk of ~1 MB per rank) are split
    // too, so their stage / fetch / gather overlap inside the call; pieces stay
    // >= 64 KiB so per-round latency does not dominate
    const size_t floor_elems = (64u << 10) / g.esz;
    const size_t want = (g.chunk + c->min_rounds - 1) / c->min_rounds;
    g.slice = std::min(g.slice, std::max(floor_elems, (want + 8 * vec - 1) / (8 * vec) * (8 * vec)));
  }
  std::vector<size_t> sizes;
  const size_t s = g.slice;
  if (c->ramp == 4 && g.chunk > s) {
    // FMX_RAMP=4: as many rounds as equal ones would take, all full slices but
    // the FIRST, which takes the remainder: the pipeline fill (every rank's
    // round-0 staging, H2D idle) shrinks without adding a round
    const size_t k = (g.chunk + s - 1) / s;
    size_t first = (g.chunk - (k - 1) * s) / vec * vec;
    if (first == 0) first = s;  // remainder under one vector: a full first round instead
    sizes.push_back(first);
    for (size_t left = g.chunk - first; left;) {
      const size_t y = std::min(s, left);
      sizes.push_back(y);
      left -= y;
    }
  } else if (c->ramp && g.chunk > s) {
    // geometric ramp s/8, s/4, s/2 up and down (as much of it as fits in half
    // the chunk each way), the middle in equal rounds of at most s
    std::vector<size_t> up;
    size_t ramp_sum = 0;
    // ramp pieces are whole vectors so every piece start stays 16-byte aligned
    // FMX_RAMP=3: one quarter-slice first round only (a short pipeline fill)
    const size_t x0 = c->ramp == 3 ? s / 4 / vec * vec : s / 8 / vec * vec;
    for (size_t x = x0; x < s && x > 0; x = x * 2 / vec * vec) {
      if (2 * (ramp_sum + x) > g.chunk) break;
      up.push_back(x);
      ramp_sum += x;
      if (c->ramp == 3) break;
    }
    const bool down = c->ramp == 1;  // FMX_RAMP=2/3: fill only, no drain ramp
    const size_t mid = g.chunk - (down ? 2 : 1) * ramp_sum;
    const size_t k = (mid + s - 1) / s;
    sizes = up;
    for (size_t i = 0; i < k; ++i) {  // equal split, multiples of the vector width
      const size_t lo = (mid * i / k) / vec * vec, hi = i + 1 == k ? mid : (mid * (i + 1) / k) / vec * vec;
      if (hi > lo) sizes.push_back(hi - lo);
    }
    if (down) sizes.insert(sizes.end(), up.rbegin(), up.rend());
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


// Reduce-scatter + all-gather through the segment, pipelined in rounds on three
// lanes: lane 0 stages (D2H), lane 1 fetches and reduces (H2D + kernel), lane 2
// gathers (H2D).  Round R uses slot R % K (K = nslots, 2 by default; the
// comments below write K = 2).  With the gather on its own lane, a rank fetches
// round R+1 while it still waits for the slowest owner of round R.
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
//      W(R-2) (every owner signalled REDUCED after its fetches of R-2).  Rounds
//      are counted across collectives and so are the waits: consecutive calls
//      may overlap on the lanes (join-stream mode, on_lanes).
//  fetch(R) of in[R%2][me][q]              -> wait STAGED(_TO)[q] >= R+1
//  reduce(R) writes out[R%2][me], last read by every q's gather(R-2):
//      W(R-1): every q signalled REDUCED >= R, which q issued after G_q(R-2).
//  gather(R) reads out[R%2][q]             -> wait REDUCED[q] >= R+1
//  in place: gather(R) overwrites piece (q, R); my stage(R) read it first,
//      because owner q's reduce(R) waited for my STAGED >= R+1.
// With FMX_LANES=2 the gather runs on lane 1 and the W/G waits are implied by
// stream order (the schedule of the first B200 runs).
enum { kEvSlotFree = 0, kEvGathered = FMX_MAX_SLOTS };  // + R % K: W(R) and G(R) above
constexpr int kEvReduceDone = 2 * FMX_MAX_SLOTS + 7;   // stage_after_reduce: reduce(R) done
// fetch lane (FMX_FETCH_LANE): F(R) fetch of round R landed in scratch slot R%2,
// S(R) reduce(R) done reading it
constexpr int kEvFetchedDev = 2 * FMX_MAX_SLOTS + 8, kEvScratchFree = kEvFetchedDev + 2;

// The all-gather of one round: wait for the owners' REDUCED, record W(R), copy
// their results out of the out-slots, record G(R).  Built per round; with
// fmx_comm_set_defer the last round's is kept (c->pending) and enqueued by the
// next collective right after its first stage, so one in-order stream stages
// bucket b+1 while peers are still reducing bucket b.  That order is valid:
// the deferred gather waits only on REDUCED flags peers signalled before their
// own next stage, and it still precedes this rank's next REDUCED signal (the
// G(R-1) wait) - the model checker runs it (FMX_TRACE_DEFER).
}  // namespace fmx
struct fmx::PendingGather {
  uint32_t R = 0;
  int LG = 0, K = 2;
  bool zc = false, coarse = true, split = false;
  int64_t scope = 0;
  std::vector<int> q;           // owners, in wait order
  std::vector<PlanSeg> segs;    // their result pieces (bytes 0: wait only)
};
namespace fmx {

static int emit_gather(fmx_comm* c, Sink& k, const PendingGather& p) {
  const int me = c->rank;
  int rc;
  const int64_t scope = k.scope();
  k.set_scope(p.scope);
  struct Restore {
    Sink& k;
    int64_t s;
    ~Restore() { k.set_scope(s); }
  } restore{k, scope};
  std::vector<PlanSeg> segs;
  if (p.coarse) {
    if ((rc = k.wait_peers(p.LG, kReduced, p.R + 1, me))) return rc;
    if ((rc = k.record(p.LG, kEvSlotFree + p.R % p.K))) return rc;  // W(R)
    for (const PlanSeg& g : p.segs)
      if (g.bytes) segs.push_back(g);
    if ((rc = k.copy(p.LG, segs, true, p.zc))) return rc;
  } else {
    for (size_t i = 0; i < p.q.size(); ++i) {
      if ((rc = k.wait_rank(p.LG, p.q[i], kReduced, p.R + 1))) return rc;
      if (!p.segs[i].bytes) continue;
      segs.assign(1, p.segs[i]);
      if ((rc = k.copy(p.LG, segs, true, p.zc))) return rc;
    }
    if ((rc = k.record(p.LG, kEvSlotFree + p.R % p.K))) return rc;  // W(R)
  }
  if (p.split && (rc = k.record(p.LG, kEvGathered + p.R % p.K))) return rc;  // G(R)
  return FMX_OK;
}

int plan_fence(fmx_comm* c, Sink& k) {
  int rc = plan_flush(c, k);
  if (rc) return rc;
  const uint32_t v = c->fence_round + 1;
  if ((rc = k.signal(kLaneMain, kFence, v)) || (rc = k.wait_peers(kLaneMain, kFence, v, c->rank)))
    return rc;
  c->fence_round = v;
  return FMX_OK;
}

void drop_pending(fmx_comm* c) {
  delete c->pending;
  c->pending = nullptr;
}

int plan_flush(fmx_comm* c, Sink& k) {
  if (!c->pending) return FMX_OK;
  PendingGather* p = c->pending;
  c->pending = nullptr;
  const int rc = emit_gather(c, k, *p);
  delete p;
  return rc;
}

// The three owner-chunk collectives share one schedule:
//   kAllreduce     stage -> fetch -> reduce (HBM + result slot) -> gather
//   kReduceScatter stage -> fetch -> reduce into recv (no result slot, no gather copies)
//   kAllgather     publish my chunk (result slot + my part of recv) -> gather
// Flags, events and slot reuse are identical, so one model-checked protocol
// covers all three.  For the last two, `count` is the per-rank count and the
// buffers follow NCCL: send/recv of reduce-scatter hold n*count / count
// elements, those of all-gather count / n*count.

int plan_allreduce(fmx_comm* c, Sink& k, const char* src, char* dst, size_t count, int dtype,
                   int op, float factor, bool aligned, int kind) {
  const int n = c->nranks, me = c->rank;
  const int LG = c->nlanes == 3 ? kLaneGather : kLaneMain;
  const int K = c->nslots;  // pipeline depth: slots per region
  const bool split = LG != kLaneMain;  // gather on its own lane: explicit W / G waits
  const bool ar = kind == kAllreduce, rs = kind == kReduceScatter, ag = kind == kAllgather;
  const Geometry g = allreduce_geometry(c, count, dtype, ar ? 0 : count);
  const bool zc = c->use_zc(g.count * g.esz);  // every rank derives the same choice
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
  // per-contributor STAGED_TO flags for this round?  FMX_GRAIN=fine: every
  // round; FMX_GRAIN=first: the first round only, so owners start fetching as
  // soon as their first contributors staged (a shorter pipeline fill)
  auto coarse_round = [&](uint32_t j) { return c->coarse && !(c->fine_first && j == 0); };

  // FMX_STAGE_ZC=1 (local knob): the stage's D2H by the SM copy kernel even on
  // the copy-engine transport, so the D2H direction carries SM stores only
  const bool szc = zc || c->stage_zc;
  // FMX_FETCH_LANE=1: the copy-engine fetch of round R+1 runs on the gather lane
  // into the other half of a double-buffered scratch while lane 1 still reduces
  // round R (with the fetch on lane 1, the fetch of R+1 queued behind reduce(R)
  // and left the H2D direction idle for the reduction's duration: two ranks per
  // GPU, r02/r3q).  Copy-engine transport, three lanes.
  const bool fl = c->fetch_lane && !zc && !ag && LG != kLaneMain;
  auto scratch_slot = [&](uint32_t R, int q) -> size_t {
    return ((fl ? (size_t)(R % 2) * n : 0) + (size_t)q) * c->slice_bytes;
  };
  // fetch(j): every contributor's piece of my chunk into HBM scratch, each as
  // soon as its contributor staged it (lane `L`)
  auto fetch = [&](uint32_t j, int L) -> int {
    const uint32_t R = R0 + j;
    const size_t mylen = g.len(me, j);
    if (fl && R >= 2 && (rc = k.wait_event(L, kEvScratchFree + R % 2))) return rc;  // S(R-2)
    if (coarse_round(j)) {
      if ((rc = k.wait_peers(L, kStaged, R + 1, me))) return rc;
      segs.clear();
      for (int q = 0; q < n && mylen; ++q) {
        if (q == me) continue;
        const size_t off = c->in_off(R, me, q);
        segs.push_back({c->at(false, off), c->scratch + scratch_slot(R, q), mylen * g.esz,
                        Annot{(int64_t)off, mylen * g.esz, q, R}, false,
                        sbuf(scratch_slot(R, q), mylen * g.esz)});
      }
      if ((rc = k.copy(L, segs, true, false))) return rc;
    } else {
      for (int i = 0; i < n - 1; ++i) {
        const int q = rot(i);
        if ((rc = k.wait_rank(L, q, kStagedTo + me, R + 1))) return rc;
        if (!mylen) continue;
        const size_t off = c->in_off(R, me, q);
        segs.clear();
        segs.push_back({c->at(false, off), c->scratch + scratch_slot(R, q), mylen * g.esz,
                        Annot{(int64_t)off, mylen * g.esz, q, R}, false,
                        sbuf(scratch_slot(R, q), mylen * g.esz)});
        if ((rc = k.copy(L, segs, true, false))) return rc;
      }
    }
    if (fl && (rc = k.record(L, kEvFetchedDev + R % 2))) return rc;  // F(R)
    return FMX_OK;
  };
  auto stage = [&](uint32_t j) -> int {
    const uint32_t R = R0 + j;
    if (ag) return FMX_OK;  // nothing to reduce: no contributions to stage
    // slot R%K was read by round R-K's fetches: W(R-K)
    if (R >= (uint32_t)K && (rc = k.wait_event(kLaneStage, kEvSlotFree + R % K))) return rc;
    if (coarse_round(j)) {  // one batch of copies, one STAGED signal
      segs.clear();
      for (int o = 0; o < n; ++o) {
        const size_t len = o == me ? 0 : g.len(o, j);
        if (!len) continue;
        const size_t off = c->in_off(R, o, me);
        segs.push_back({src + g.lo(o, j) * g.esz, c->at(szc, off), len * g.esz,
                        Annot{(int64_t)off, len * g.esz, me, R}, true,
                        ubuf(g.lo(o, j) * g.esz, len * g.esz)});
      }
      return k.copy_signal(kLaneStage, segs, false, szc, kStaged, R + 1);
    }
    for (int i = 0; i < n - 1; ++i) {
      const int o = rot(i);
      const size_t len = g.len(o, j);
      segs.clear();
      if (len) {
        const size_t off = c->in_off(R, o, me);
        segs.push_back({src + g.lo(o, j) * g.esz, c->at(szc, off), len * g.esz,
                        Annot{(int64_t)off, len * g.esz, me, R}, true,
                        ubuf(g.lo(o, j) * g.esz, len * g.esz)});
        if ((rc = k.copy(kLaneStage, segs, false, szc))) return rc;
      }
      if ((rc = k.signal(kLaneStage, kStagedTo + o, R + 1))) return rc;
    }
    return FMX_OK;
  };

  // a deferred gather of the previous allreduce goes after this call's first
  // stage(s) (allreduce) or first of all (reduce-scatter / all-gather)
  if (!ar && (rc = plan_flush(c, k))) return rc;
  // lane 0 stages K-1 rounds ahead of the reduction (stage_after_reduce: stage
  // j+K-1 is enqueued after reduce(j) and waits for it on the GPU)
  const uint32_t ahead = (uint32_t)K - 1;
  const bool sar = c->stage_after_reduce && !ag;
  for (uint32_t j = 0; j < ahead && j < g.rounds; ++j)
    if ((rc = stage(j))) return rc;
  if ((rc = plan_flush(c, k))) return rc;
  if (fl && (rc = fetch(0, LG))) return rc;
  for (uint32_t j = 0; j < g.rounds; ++j) {
    const uint32_t R = R0 + j;
    if (!sar && j + ahead < g.rounds && (rc = stage(j + ahead))) return rc;
    if (fl && j + 1 < g.rounds && (rc = fetch(j + 1, LG))) return rc;
    // lane 1: fetch, then reduce-scatter my chunk in ascending rank order
    const size_t mylen = g.len(me, j);
    if (mylen && ag) {
      // publish: my piece into my result slot (and into my part of recv)
      const size_t out_off = c->out_off(R, me);
      if (split && R + 1 >= (uint32_t)K && (rc = k.wait_event(kLaneMain, kEvSlotFree + (R + 1 - K) % K)))
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
      if (ar && c->sgd) {   // fused SGD step on my piece of the parameters (fp32)
        const SgdEpi& e = *c->sgd;
        a.sgd = 1;
        a.mom = e.mom ? e.mom + g.start[j] * g.esz : nullptr;
        a.lr = e.lr;
        a.mu = e.mu;
        a.damp = e.damp;
        a.wd = e.wd;
        a.nesterov = e.nesterov;
        a.init = e.init;
      }
      const size_t out_off = c->out_off(R, me);
      pr.user_rw = ubuf(g.lo(me, j) * g.esz, mylen * g.esz);
      // result slot by the copy engine: FMX_RESULT_VIA_CE, or with the fetch lane on
      // long pipelines (two ranks per GPU, >= rce_rounds rounds: the SM result store
      // starves under the copy engines' D2H, a copy-engine write does not - 1 GiB
      // 48.2-49.4 vs 53.7-54.5 ms; at 2 rounds the extra copy costs more, r02/r3t).
      // A local choice: peers only see REDUCED.
      const bool via_ce = ar && !zc && (c->result_via_ce || (fl && g.rounds >= (uint32_t)c->rce_rounds));
      if (ar && !via_ce) {
        a.out_sys = c->at(true, out_off);
        pr.write = Annot{(int64_t)out_off, mylen * g.esz, me, R};
      }
      // each contribution is fetched as soon as its contributor staged it
      // (fetch lane: already enqueued on lane LG; wait for it here)
      if (fl) {
        if ((rc = k.wait_event(kLaneMain, kEvFetchedDev + R % 2))) return rc;  // F(R)
      } else if (!zc) {
        if ((rc = fetch(j, kLaneMain))) return rc;
      } else if (coarse_round(j)) {   // zero-copy: the reduction reads the slots itself
        if ((rc = k.wait_peers(kLaneMain, kStaged, R + 1, me))) return rc;
      } else {
        for (int i = 0; i < n - 1; ++i)
          if ((rc = k.wait_rank(kLaneMain, rot(i), kStagedTo + me, R + 1))) return rc;
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
          a.src[q] = c->scratch + scratch_slot(R, q);
          pr.scratch_reads.push_back(sbuf(scratch_slot(R, q), mylen * g.esz));
        }
      }
      // out[R%K][me] is free once every peer gathered round R-K: W(R-K+1)
      if (split && R + 1 >= (uint32_t)K && (rc = k.wait_event(kLaneMain, kEvSlotFree + (R + 1 - K) % K)))
        return rc;
      if ((rc = k.reduce(kLaneMain, pr))) return rc;
      if (fl && (rc = k.record(kLaneMain, kEvScratchFree + R % 2))) return rc;  // S(R)
      if (sar && j + ahead < g.rounds && (rc = k.record(kLaneMain, kEvReduceDone))) return rc;
      if (via_ce) {  // result slot written by the copy engine from HBM
        segs.clear();
        segs.push_back({my_out(j), c->at(false, out_off), mylen * g.esz,
                        Annot{(int64_t)out_off, mylen * g.esz, me, R}, true,
                        ubuf(g.lo(me, j) * g.esz, mylen * g.esz)});
        if ((rc = k.copy(kLaneMain, segs, false, false))) return rc;
      }
    }
    if (sar && j + ahead < g.rounds) {
      if (mylen && (rc = k.wait_event(kLaneStage, kEvReduceDone))) return rc;
      if ((rc = stage(j + ahead))) return rc;
    }
    // REDUCED(R) also says "my gather(R-1) is done": G(R-1)
    if (split && R >= 1 && (rc = k.wait_event(kLaneMain, kEvGathered + (R - 1) % K))) return rc;
    if ((rc = k.signal(kLaneMain, kReduced, R + 1))) return rc;
    // all-gather (lane LG): each owner's result as soon as that owner has it
    PendingGather pg;
    pg.R = R;
    pg.LG = LG;
    pg.K = K;
    pg.zc = zc;
    pg.coarse = c->coarse_gather;
    pg.split = split;
    pg.scope = k.scope();
    for (int i = 0; i < n - 1; ++i) {
      // coarse: ascending owners, one copy batch; fine: rotated, a wait per owner
      const int q = pg.coarse ? (i < me ? i : i + 1) : rot(i);
      const size_t len = rs ? 0 : g.len(q, j);
      const size_t off = c->out_off(R, q);
      pg.q.push_back(q);
      pg.segs.push_back({c->at(zc, off), dst + g.lo(q, j) * g.esz, len * g.esz,
                         Annot{(int64_t)off, len * g.esz, q, R}, false,
                         ubuf(g.lo(q, j) * g.esz, len * g.esz)});
    }
    if (ar && c->defer_gather && j + 1 == g.rounds) {
      c->pending = new PendingGather(std::move(pg));  // enqueued by the next call / fmx_comm_flush
    } else if ((rc = emit_gather(c, k, pg))) {
      return rc;
    }
  }
  c->ar_round += g.rounds;
  return FMX_OK;
}

// One-shot allreduce for small messages (AUTO / ZC, bytes <= oneshot_max): the
// two-hop reduce-scatter / all-gather above pays STAGED -> REDUCED -> gather,
// three flag hops and five launches, for a message the link moves in a few
// microseconds.  Here every rank publishes its whole buffer into its one-shot
// slot with one zero-copy kernel that releases OS_READY itself, waits for every
// peer's OS_READY, and reduces all n contributions in ascending rank order
// straight out of the segment (its own from HBM) into its buffer: one flag hop,
// two launches, one flag write, and every rank computes the same bits as the owner of that
// chunk would (same kernel, same order).  Single lane (lane 1), no HBM scratch.
// Slots alternate (kOsSlots = 2) and need no credit flag: slot J % 2 is next
// written at call J + 2, after this rank's wait of call J + 1 saw every peer's
// OS_READY >= J + 2 - and each peer publishes call J + 1 only after its reduce
// of call J (which read my slot) in its stream order.  The model checker
// confirms it (tests/test_protocol_model.py).  Own round counter and flag:
// mixing with the pipelined collectives shares nothing but the stream.
constexpr uint32_t kOsTag = 1u << 30;  // trace: one-shot rounds, apart from pipeline rounds

int plan_allreduce_oneshot(fmx_comm* c, Sink& k, const char* src, char* dst, size_t count,
                           int dtype, int op, float factor, bool aligned) {
  const int n = c->nranks, me = c->rank;
  const size_t esz = dtype == FMX_FLOAT32 ? 4 : 2, bytes = count * esz;
  const uint32_t J = c->os_round;
  int rc;
  if ((rc = plan_flush(c, k))) return rc;
  const size_t mine = c->os_slot_off(J, me);
  std::vector<PlanSeg> segs{{src, c->at(true, mine), bytes, Annot{(int64_t)mine, bytes, me, J | kOsTag},
                             true, ubuf(0, bytes)}};
  if ((rc = k.copy_signal(kLaneMain, segs, false, true, kOsReady, J + 1))) return rc;
  PlanReduce pr;
  memset(&pr.args, 0, sizeof pr.args);
  pr.dtype = dtype;
  pr.aligned = aligned;
  pr.args.nsrc = n;
  pr.args.len = count;
  pr.args.op = op;
  pr.args.factor = factor;
  pr.args.out_dev = dst;
  pr.user_rw = ubuf(0, bytes);
  for (int q = 0; q < n; ++q) {
    if (q == me) {
      pr.args.src[q] = src;
      continue;
    }
    const size_t off = c->os_slot_off(J, q);
    pr.args.src[q] = c->at(true, off);
    pr.args.sys_mask |= 1ull << q;
    pr.reads.push_back(Annot{(int64_t)off, bytes, q, J | kOsTag});
  }
  // wait for every peer's publish, then reduce (fused into one kernel for MPS ranks)
  if ((rc = k.wait_reduce(kLaneMain, pr, kOsReady, J + 1, me))) return rc;
  c->os_round = J + 1;
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
  if ((rc = plan_flush(c, k))) return rc;
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
  const size_t esz = dtype == FMX_FLOAT32 ? 4 : 2;
  const bool zc = c->use_zc(count * esz);
  const size_t bslice = (size_t)c->nranks * c->slice_bytes / esz;
  const uint32_t rounds = (uint32_t)((count + bslice - 1) / bslice);
  std::vector<PlanSeg> segs(1);
  int rc;
  if ((rc = plan_flush(c, k))) return rc;
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

}  // namespace fmx

using namespace fmx;

extern "C" {

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
  c.transport = (transport == FMX_TRANSPORT_ZC || transport == FMX_TRANSPORT_AUTO) ? transport
                                                                                  : FMX_TRANSPORT_CE;
  apply_proto(&c, proto_from_env());
  // FMX_TRACE_DEFER=1: fmx_comm_set_defer (an allreduce's last gather deferred)
  c.defer_gather = getenv("FMX_TRACE_DEFER") && atoi(getenv("FMX_TRACE_DEFER"));
  c.stage_after_reduce = getenv("FMX_STAGE_AFTER_REDUCE") && atoi(getenv("FMX_STAGE_AFTER_REDUCE"));
  if (const char* v = getenv("FMX_FETCH_LANE")) c.fetch_lane = atoi(v) != 0;
  if (const char* v = getenv("FMX_RCE_ROUNDS")) c.rce_rounds = std::max(1, atoi(v));
  c.slice_bytes = slice_bytes;
  size_t max_bytes = 0;
  for (int i = 0; i < nops; ++i) max_bytes = std::max(max_bytes, counts[i] * (dtypes[i] ? 2 : 4));
  c.L = compute_layout(nranks, c.nslots, slice_bytes, max_bytes, c.oneshot_max);
  c.total_bytes = c.L.total;
  std::string out;
  TraceSink sink(&out);
  sink.nranks = nranks;
  // fake user buffers: only their offsets matter and they never reach SHM
  static char dummy[16] __attribute__((aligned(16)));
  // FMX_TRACE_OVERLAP=1: the join-stream mode - consecutive device-buffer
  // collectives (distinct buffers) are not separated by a join on the lanes;
  // host-path calls and broadcasts still are (on_lanes' barrier)
  const bool overlap = getenv("FMX_TRACE_OVERLAP") && atoi(getenv("FMX_TRACE_OVERLAP"));
  auto device_class = [&](int i) {
    return kinds[i] == 0 || kinds[i] == 3 || kinds[i] == 4 || kinds[i] == 5;
  };
  // FMX_TRACE_REPLAYS=k: the op list is a captured graph, launched k times
  // (fmx_graph_*): every replay runs the captured schedule - same slots, same
  // rounds - with flag values re-based by the counters' advance, ends with the
  // fence capture_end appends (FMX_TRACE_REPLAY_FENCE=0 drops it: the checker
  // must then object), and sees no event of another replay
  const int replays = getenv("FMX_TRACE_REPLAYS") ? std::max(1, atoi(getenv("FMX_TRACE_REPLAYS"))) : 0;
  const bool replay_fence = !getenv("FMX_TRACE_REPLAY_FENCE") || atoi(getenv("FMX_TRACE_REPLAY_FENCE"));
  uint32_t c0[kNumCounters], delta[kNumCounters] = {};
  for (int k = 0; k < kNumCounters; ++k) c0[k] = *c.counter(k);
  for (int rep = 0; rep < std::max(1, replays); ++rep) {
  if (replays && rep > 0) {
    for (int k = 0; k < kNumCounters; ++k) {
      *c.counter(k) = c0[k];
      sink.flag_off[k] = (uint32_t)rep * delta[k];
    }
    sink.round_tag = (uint32_t)rep << 24;
    sink.epoch = rep;
  }
  for (int i = 0; i < nops; ++i) {
    int rc;
    if (!overlap || i == 0 || !device_class(i) || !device_class(i - 1)) sink.join();
    sink.user_base = overlap ? (int64_t)i << 40 : 0;
    if (kinds[i] == 1 && (!roots || roots[i] < 0 || roots[i] >= nranks))
      return fail(FMX_ERR_INVALID_ARG, "bad broadcast root");
    const size_t esz = dtypes[i] ? 2 : 4;
    if (kinds[i] == 5)  // fmx_comm_flush
      rc = plan_flush(&c, sink);
    else if (kinds[i] == 0 && c.use_oneshot(counts[i] * esz))
      rc = plan_allreduce_oneshot(&c, sink, dummy, dummy, counts[i], dtypes[i], FMX_OP_SUM, 1.0f, true);
    else if (kinds[i] == 0)
      rc = plan_allreduce(&c, sink, dummy, dummy, counts[i], dtypes[i], FMX_OP_SUM, 1.0f, true);
    else if (kinds[i] == 3 || kinds[i] == 4)  // reduce-scatter / all-gather, in place
      rc = plan_allreduce(&c, sink, dummy, dummy, counts[i], dtypes[i], FMX_OP_SUM, 1.0f, true,
                          kinds[i] == 3 ? kReduceScatter : kAllgather);
    else if (kinds[i] == 2)
      rc = plan_allreduce_host(&c, sink, 0, counts[i], dtypes[i], FMX_OP_SUM, 1.0f);
    else
      rc = plan_broadcast(&c, sink, dummy, dummy, counts[i], dtypes[i], roots ? roots[i] : 0);
    if (rc) {
      drop_pending(&c);
      return rc;
    }
  }
  if (replays) {
    if (c.pending) {
      drop_pending(&c);
      return fail(FMX_ERR_INVALID_ARG, "captured sequence ends with a deferred gather");
    }
    sink.join();  // the fence node depends on every leaf of the graph
    if (replay_fence && plan_fence(&c, sink)) return FMX_ERR_INVALID_ARG;
    if (rep == 0)
      for (int k = 0; k < kNumCounters; ++k) delta[k] = *c.counter(k) - c0[k];
  }
  }
  if (c.pending) {  // an unflushed deferred gather: the sequence must end with a flush
    drop_pending(&c);
    return fail(FMX_ERR_INVALID_ARG, "deferred gather not flushed (end the sequence with kind 5)");
  }
  sink.join();
  if (used) *used = out.size() + 1;
  if (!buf || cap < out.size() + 1) return fail(FMX_ERR_INVALID_ARG, "trace buffer too small");
  memcpy(buf, out.c_str(), out.size() + 1);
  return FMX_OK;
}

}  // extern "C"

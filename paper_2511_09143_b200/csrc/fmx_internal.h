// Internal declarations shared by the host and device halves of libflexshm.
#pragma once

#include <atomic>
#include <cstddef>
#include <cstdint>
#include <string>

#include "../../include/flexshm.h"

namespace fmx {

// ---- error state (thread-local, fmx_last_error / fmx_dup_ranks) ------------
int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
void set_dup(int a, int b);

// ---- SHM segment layout ----------------------------------------------------
// [header 4 KiB][peer table][flag lines][AR in-slots][AR out-slots][BC slots]
// [one-shot slots][user region of rank 0] ... [user region of rank n-1]
// Every region starts on a 4 KiB boundary; every flag owns a 64-byte line.
constexpr uint32_t kMagicReady = 0x464D5831u;  // "FMX1"
constexpr uint32_t kVersion = 3;
// Per rank: 8 scalar flags, then one STAGED_TO flag per destination owner.
// OS_READY is the one-shot small-message allreduce's own round counter
// (plan_allreduce_oneshot, flexshm_plan.cpp); FENCE the end-of-replay fence of
// captured graphs (fmx_graph_*, flexshm_comm.cu).
enum Flag { kStaged = 0, kReduced = 1, kBcStaged = 2, kBcDone = 3, kOsReady = 4, kFence = 5,
            kStagedTo = 8 };
// One-shot slots: [kOsSlots][rank][os_bytes], alternating between calls.
constexpr int kOsSlots = 2;
constexpr size_t kOneShotCap = 1u << 20;  // largest one-shot message (FMX_ONESHOT_MAX is clamped)
constexpr int kFlagsPerRank = kStagedTo + FMX_MAX_RANKS;

struct alignas(64) PeerSlot {
  std::atomic<int32_t> state;  // 0 empty, 1 published
  int32_t pid;
  fmx_peer_info info;
};

// Settings that change the schedule - piece boundaries, which flags are
// signalled, which lane gathers, the transport of a collective.  Rank 0
// publishes its own (read from its environment, FMX_RAMP, FMX_MIN_ROUNDS,
// FMX_GRAIN, FMX_GATHER_GRAIN, FMX_LANES, FMX_RESULT_VIA_CE, FMX_ZC_MAX,
// FMX_ONESHOT_MAX) in the
// segment header and every rank adopts them, so ranks cannot disagree on the
// protocol (a mismatch would give wrong results or park a stream forever).
struct Proto {
  int32_t ramp, min_rounds, coarse, fine_first, coarse_gather, nlanes, result_via_ce;
  int32_t oneshot_max;  // bytes; allreduces up to this size take the one-shot path (0: off)
  uint64_t zc_max;
};

struct Header {
  std::atomic<uint32_t> magic;
  uint32_t version;
  int32_t nranks;
  int32_t nslots;
  uint64_t slice_bytes;
  uint64_t total_bytes;
  uint64_t peers_off, flags_off, ar_in_off, ar_out_off, bc_off, os_off, os_bytes;
  uint64_t user_off, user_bytes;  // per-rank registered host buffers
  int32_t creator_pid;
  int32_t mig_aware;
  alignas(64) std::atomic<int32_t> arrived;
  alignas(64) std::atomic<int32_t> mapped;
  alignas(64) std::atomic<int32_t> aborted;
  alignas(64) std::atomic<int64_t> barrier_count;
  alignas(64) std::atomic<int32_t> departed;
  alignas(64) std::atomic<int32_t> touched;  // ranks done first-touching their regions
  char job_key[128];
  Proto proto;  // rank 0's schedule settings, adopted by every rank
};

static_assert(sizeof(Header) <= 4096, "the header owns the first page of the segment");

struct Layout {
  size_t peers_off, flags_off, ar_in_off, ar_out_off, bc_off, os_off, os_bytes, user_off, user_bytes,
      total;
};
Layout compute_layout(int nranks, int nslots, size_t slice_bytes, size_t user_bytes,
                      size_t os_bytes);

inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

double now_s();

}  // namespace fmx

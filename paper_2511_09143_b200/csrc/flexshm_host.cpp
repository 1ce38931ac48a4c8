// Host half of libflexshm: error state and the bootstrap rules of the
// reference's communicator layer, applied to fixed-size C records.
//
//   fmx_check_peer      <- PeerInfo.__post_init__   (commsim.py:35-42)
//   fmx_validate_peers  <- discover_peers           (commsim.py:67-88)
//   fmx_topology        <- build_topology           (commsim.py:91-116)
//   fmx_restore_bus_id  <- restore_bus_id           (commsim.py:119-123)
//
// No CUDA in this file: everything here runs (and is tested) without a GPU.
#include <algorithm>
#include <cctype>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "fmx_internal.h"

namespace fmx {

static thread_local char g_err[512] = "";
static thread_local int g_dup_a = -1, g_dup_b = -1;

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return code;
}

void set_dup(int a, int b) {
  g_dup_a = a;
  g_dup_b = b;
}

double now_s() {
  using namespace std::chrono;
  return duration<double>(steady_clock::now().time_since_epoch()).count();
}

Layout compute_layout(int nranks, int nslots, size_t slice_bytes, size_t user_bytes,
                      size_t os_bytes) {
  Layout L;
  const size_t page = 4096;
  size_t off = page;  // header
  L.peers_off = off;
  off = align_up(off + sizeof(PeerSlot) * nranks, page);
  L.flags_off = off;
  off = align_up(off + (size_t)64 * kFlagsPerRank * nranks, page);
  L.ar_in_off = off;
  off += (size_t)nslots * nranks * nranks * slice_bytes;
  L.ar_out_off = off;
  off += (size_t)nslots * nranks * slice_bytes;
  L.bc_off = off;
  off += (size_t)nslots * nranks * slice_bytes;
  L.os_off = off = align_up(off, page);
  L.os_bytes = align_up(os_bytes, page);
  off += (size_t)kOsSlots * nranks * L.os_bytes;
  L.user_off = off = align_up(off, page);
  L.user_bytes = align_up(user_bytes, page);
  off += (size_t)nranks * L.user_bytes;
  L.total = align_up(off, page);
  return L;
}

// "XX:XX:XX.d" with upper-case hex; digit d must be 0 when canonical_only.
// Like Python's re.match with a trailing `$`, one final '\n' is tolerated.
static bool match_label(const char* s, bool canonical_only) {
  size_t len = strnlen(s, FMX_BUS_ID_LEN);
  if (!(len == 10 || (len == 11 && s[10] == '\n'))) return false;
  for (int i = 0; i < 10; ++i) {
    char c = s[i];
    if (i == 2 || i == 5) {
      if (c != ':') return false;
    } else if (i == 8) {
      if (c != '.') return false;
    } else if (i == 9) {
      if (canonical_only ? c != '0' : !(c >= '0' && c <= '9')) return false;
    } else if (!((c >= '0' && c <= '9') || (c >= 'A' && c <= 'F'))) {
      return false;
    }
  }
  return true;
}

static void upper_copy(char* dst, const char* src, size_t cap) {
  size_t i = 0;
  for (; i + 1 < cap && src[i]; ++i) dst[i] = (char)toupper((unsigned char)src[i]);
  dst[i] = 0;
}

}  // namespace fmx

using namespace fmx;

extern "C" {

int fmx_abi_version(void) { return FMX_ABI_VERSION; }

const char* fmx_last_error(void) { return g_err; }

int fmx_dup_ranks(int* rank_a, int* rank_b) {
  if (rank_a) *rank_a = g_dup_a;
  if (rank_b) *rank_b = g_dup_b;
  return g_dup_a >= 0 ? FMX_OK : FMX_ERR_INVALID_ARG;
}

int fmx_check_peer(fmx_peer_info* p) {
  if (!p) return fail(FMX_ERR_INVALID_ARG, "null peer");
  char up[FMX_BUS_ID_LEN];
  if (memchr(p->pcie_bus_id, 0, FMX_BUS_ID_LEN) == nullptr)
    return fail(FMX_ERR_MALFORMED_LABEL, "bus id is not NUL-terminated");
  upper_copy(up, p->pcie_bus_id, sizeof up);
  if (!match_label(up, true))
    return fail(FMX_ERR_MALFORMED_LABEL, "bus id '%s' is not a canonical device id",
                p->pcie_bus_id);
  memset(p->pcie_bus_id, 0, FMX_BUS_ID_LEN);
  memcpy(p->pcie_bus_id, up, strlen(up));
  if (memchr(p->mig_id, 0, FMX_MIG_ID_LEN) == nullptr)
    return fail(FMX_ERR_INVALID_ARG, "mig_id is not NUL-terminated");
  if (p->mig_id[0] == 0) return fail(FMX_ERR_EMPTY_MIG_ID, "rank %d has an empty mig_id", p->rank);
  return FMX_OK;
}

int fmx_validate_peers(const fmx_peer_info* peers, int n, int mig_aware, int* rank_a,
                       int* rank_b) {
  if (n < 0 || (n > 0 && !peers)) return fail(FMX_ERR_INVALID_ARG, "bad peer array");
  // ranks must be exactly 0..n-1
  std::vector<int> at(n, -1);
  for (int i = 0; i < n; ++i) {
    int r = peers[i].rank;
    if (r < 0 || r >= n || at[r] != -1)
      return fail(FMX_ERR_BAD_RANKS, "ranks must be 0..%d and distinct", n - 1);
    at[r] = i;
  }
  // first collision in ascending rank order -> (holder, newcomer)
  std::map<std::tuple<int64_t, std::string, std::string>, int> holder;
  for (int r = 0; r < n; ++r) {
    const fmx_peer_info& p = peers[at[r]];
    std::string bus(p.pcie_bus_id, strnlen(p.pcie_bus_id, FMX_BUS_ID_LEN));
    std::string mig = mig_aware ? std::string(p.mig_id, strnlen(p.mig_id, FMX_MIG_ID_LEN))
                                : std::string();
    auto key = std::make_tuple(p.host_hash, bus, mig);
    auto it = holder.find(key);
    if (it != holder.end()) {
      set_dup(it->second, r);
      if (rank_a) *rank_a = it->second;
      if (rank_b) *rank_b = r;
      return fail(FMX_ERR_DUPLICATE_DEVICE, "ranks %d and %d resolve to the same device",
                  it->second, r);
    }
    holder.emplace(key, r);
  }
  return FMX_OK;
}

int fmx_topology(const fmx_peer_info* peers, int n, char* labels, char* mig_buses,
                 int* mig_counts, int* n_buses) {
  if (n < 0 || (n > 0 && (!peers || !labels))) return fail(FMX_ERR_INVALID_ARG, "bad args");
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(),
                   [&](int a, int b) { return peers[a].rank < peers[b].rank; });
  std::vector<std::string> buses;
  std::vector<int> counts;
  for (int k = 0; k < n; ++k) {
    const fmx_peer_info& p = peers[order[k]];
    std::string bus(p.pcie_bus_id, strnlen(p.pcie_bus_id, FMX_BUS_ID_LEN));
    int idx = -1;
    for (size_t b = 0; b < buses.size(); ++b)
      if (buses[b] == bus) idx = (int)b;
    int ordinal = idx < 0 ? 0 : counts[idx];
    if (ordinal >= FMX_MAX_RANKS_PER_BUS)
      return fail(FMX_ERR_MALFORMED_LABEL,
                  "more than 10 ranks on bus %s; ordinal does not fit one digit", bus.c_str());
    std::string label = bus;
    if (ordinal > 0 && !label.empty()) label.back() = (char)('0' + ordinal);
    char* dst = labels + (size_t)k * FMX_BUS_ID_LEN;
    memset(dst, 0, FMX_BUS_ID_LEN);
    memcpy(dst, label.data(), std::min(label.size(), (size_t)FMX_BUS_ID_LEN - 1));
    if (idx < 0) {
      buses.push_back(bus);
      counts.push_back(1);
    } else {
      counts[idx]++;
    }
  }
  if (n_buses) *n_buses = (int)buses.size();
  for (size_t b = 0; b < buses.size(); ++b) {
    if (mig_buses) {
      char* dst = mig_buses + b * FMX_BUS_ID_LEN;
      memset(dst, 0, FMX_BUS_ID_LEN);
      memcpy(dst, buses[b].data(), std::min(buses[b].size(), (size_t)FMX_BUS_ID_LEN - 1));
    }
    if (mig_counts) mig_counts[b] = counts[b];
  }
  return FMX_OK;
}

int fmx_restore_bus_id(const char* label, char* out) {
  if (!label || !out) return fail(FMX_ERR_INVALID_ARG, "null label");
  char up[FMX_BUS_ID_LEN + 8];
  if (strnlen(label, sizeof up) >= sizeof up)
    return fail(FMX_ERR_MALFORMED_LABEL, "bad bus id label");
  upper_copy(up, label, sizeof up);
  if (!match_label(up, false)) return fail(FMX_ERR_MALFORMED_LABEL, "bad bus id label '%s'", label);
  // label.upper()[:-1] + "0"
  size_t len = strlen(up);
  memset(out, 0, FMX_BUS_ID_LEN);
  memcpy(out, up, len - 1);
  out[len - 1] = '0';
  return FMX_OK;
}

}  // extern "C"

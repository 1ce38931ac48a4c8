// ThreadSanitizer harness for the host half of libflexshm: the SHM bootstrap
// (segment creation, peer-table publication, arrival counters, first-touch
// barrier), fmx_barrier and fmx_comm_abort, with every rank a thread of one
// process (TSAN sees threads, not processes).  FMX_TRANSPORT_HOST makes no CUDA
// call, so this runs without a GPU.  Build + run: tools/sanitize/run_tsan.sh.
// Scope: every rank maps the segment itself (its own virtual addresses), so
// TSAN checks the process-wide state (call_once driver loading, thread-local
// error state, the communicator objects) and each rank's own accesses, not
// cross-rank accesses to the segment - those are the protocol the model
// checker covers (tests/test_protocol_model.py) and the atomics of Header.
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/flexshm.h"

static int run_job(int n, const char* key, int barriers, bool abort_mid) {
  std::vector<int> rc(n, -1);
  std::vector<std::thread> th;
  for (int r = 0; r < n; ++r)
    th.emplace_back([&, r] {
      fmx_peer_info p;
      memset(&p, 0, sizeof p);
      p.rank = r;
      snprintf(p.pcie_bus_id, sizeof p.pcie_bus_id, "%02X:00:00.0", 0x1b + r / 7);
      snprintf(p.mig_id, sizeof p.mig_id, "MIG-tsan-%d", r);
      p.host_hash = 42;
      p.pid_hash = 1000 + r;
      fmx_comm_t c = nullptr;
      int e = fmx_comm_init(&c, key, n, r, &p, 1, 0, 0, 1 << 16, FMX_TRANSPORT_HOST, 30.0);
      if (e) {
        rc[r] = e;
        return;
      }
      for (int b = 0; b < barriers && !e; ++b) {
        if (abort_mid && r == n - 1 && b == barriers / 2) {
          fmx_comm_abort(c);
          e = FMX_ERR_ABORTED;
          break;
        }
        e = fmx_barrier(c, 30.0);
      }
      void* buf = nullptr;
      size_t bytes = 0;
      if (fmx_host_buffer(c, r, &buf, &bytes) == FMX_OK && buf) memset(buf, r, 64);
      fmx_comm_destroy(c);
      rc[r] = e;
    });
  for (auto& t : th) t.join();
  int bad = 0;
  for (int r = 0; r < n; ++r)
    if (rc[r] != FMX_OK && !(abort_mid && rc[r] == FMX_ERR_ABORTED)) ++bad;
  printf("job %s: %d ranks, %d barriers%s: %d rank(s) failed\n", key, n, barriers,
         abort_mid ? ", abort midway" : "", bad);
  return bad;
}

int main() {
  int bad = 0;
  bad += run_job(2, "tsan-a", 50, false);
  bad += run_job(7, "tsan-b", 50, false);
  bad += run_job(14, "tsan-c", 20, false);
  bad += run_job(7, "tsan-d", 20, true);
  return bad ? 1 : 0;
}

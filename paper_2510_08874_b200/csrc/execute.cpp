// Whole-multiply launch through the C-ABI: um_execute / um_sync_all.
//
// Replaces the reference's driver loop
//   runtime.execute_multiply (runtime.py:339-387): every rank's run_direct,
//   the run-level barrier, then reduce_replicas(0) when C is replicated
// for a caller that is not Python.  The host planner (opgen/schedule/engine,
// or any other front end) serialises each rank's issue plan -- copy-engine
// pulls, prepared K1 launches (um_gemm_prepare handles that carry the
// in-kernel pulls, k-chains and completion slots), the waits between them --
// and the replica reduction steps; um_execute replays all of it
// asynchronously on library-owned streams (one compute and one get stream
// per rank, one reduce stream per device) with no host synchronisation, and
// um_sync_all is the host-side barrier.
//
// Ordering (SPEC.md:586-594 restated on streams):
//   * every stream of this call starts after all work of the previous
//     um_execute on the same devices (per-device "tail" events);
//   * a launch that reads a copy-engine pull waits for that pull's event
//     (action UM_ACT_WAIT_COPY);
//   * reduction steps start after every rank's last action (the reference's
//     run-level barrier before reduce_replicas).
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "um_internal.h"

namespace um {
namespace {

struct Streams {
  std::map<std::pair<int, int>, cudaStream_t> rank_streams;   // (rank, role) -> stream
  std::map<int, cudaStream_t> reduce_streams;                 // device -> stream
  std::map<int, cudaEvent_t> tail;                            // device -> last event of the last execute
  std::mutex mu;
};

Streams& S() {
  static Streams* s = new Streams();   // never destroyed: streams outlive static teardown order
  return *s;
}

int stream_for(std::map<std::pair<int, int>, cudaStream_t>& m, int rank, int role, int device, cudaStream_t* out) {
  auto key = std::make_pair(rank, role);
  auto it = m.find(key);
  if (it != m.end()) {
    *out = it->second;
    return UM_OK;
  }
  DeviceGuard g(device);
  cudaStream_t s;
  UM_CUDA_CHECK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  m[key] = s;
  *out = s;
  return UM_OK;
}

int event_on(cudaStream_t s, int device, cudaEvent_t* out) {
  DeviceGuard g(device);
  UM_CUDA_CHECK(cudaEventCreateWithFlags(out, cudaEventDisableTiming));
  UM_CUDA_CHECK(cudaEventRecord(*out, s));
  return UM_OK;
}

}  // namespace
}  // namespace um

using namespace um;

extern "C" int um_execute(const um_rank_plan* ranks, int32_t nranks, const um_reduce_step* reduces, int32_t nreduce,
                          const um_exec_cfg* cfg) {
  if (nranks < 0 || (nranks > 0 && !ranks) || nreduce < 0 || (nreduce > 0 && !reduces))
    return fail(UM_EVALUE, "um_execute: bad plan arrays");
  if (cfg && (cfg->prefetch_depth < 1 || cfg->max_inflight_gemms < 1 || cfg->max_inflight_accums < 1))
    return fail(UM_EVALUE, "ExecConfig counts must be >= 1");   // runtime.py:35-37
  Streams& st = S();
  std::lock_guard<std::mutex> lk(st.mu);
  struct Range {   // NVTX range "um:um_execute" around the whole host issue
    Range() { nvtxRangePushA("um:um_execute"); }
    ~Range() { nvtxRangePop(); }
  } range;
  int rc;
  std::vector<cudaEvent_t> events;       // destroyed at the end (recorded work keeps running)
  auto cleanup = [&]() {
    for (cudaEvent_t e : events) cudaEventDestroy(e);
  };
  // per-device start: previous execute's tail
  std::map<int, cudaEvent_t> start = st.tail;
  std::vector<cudaEvent_t> rank_done;
  std::map<int, std::vector<cudaEvent_t>> dev_done;
  for (int r = 0; r < nranks; ++r) {
    const um_rank_plan& P = ranks[r];
    if (P.ncopies < 0 || (P.ncopies > 0 && !P.copies) || P.nactions < 0 || (P.nactions > 0 && !P.actions)) {
      cleanup();
      return fail(UM_EVALUE, "um_execute: rank " + std::to_string(P.rank) + ": bad copy / action arrays");
    }
    DeviceGuard g(P.device);
    cudaStream_t cs, gs;
    if ((rc = stream_for(st.rank_streams, P.rank, 0, P.device, &cs)) ||
        (rc = stream_for(st.rank_streams, P.rank, 1, P.device, &gs))) {
      cleanup();
      return rc;
    }
    for (auto& kv : start) {
      if (cudaStreamWaitEvent(cs, kv.second, 0) != cudaSuccess || cudaStreamWaitEvent(gs, kv.second, 0) != cudaSuccess) {
        cleanup();
        return fail(UM_ECUDA, "cudaStreamWaitEvent (start)");
      }
    }
    // copy-engine pulls first, in first-use order, each with its arrival event
    std::vector<cudaEvent_t> copy_ev(P.ncopies, nullptr);
    for (int i = 0; i < P.ncopies; ++i) {
      if ((rc = um_get(&P.copies[i].src, &P.copies[i].dst, gs))) {
        cleanup();
        return rc;
      }
      if ((rc = event_on(gs, P.device, &copy_ev[i]))) {
        cleanup();
        return rc;
      }
      events.push_back(copy_ev[i]);
    }
    std::vector<char> waited(P.ncopies, 0);
    for (int a = 0; a < P.nactions; ++a) {
      const um_exec_action& act = P.actions[a];
      if (act.kind == UM_ACT_LAUNCH) {
        if ((rc = um_gemm_launch(act.handle, cs))) {
          cleanup();
          return rc;
        }
      } else if (act.kind == UM_ACT_WAIT_COPY) {
        if (act.arg < 0 || act.arg >= P.ncopies) {
          cleanup();
          return fail(UM_EVALUE, "um_execute: wait on a copy outside the rank's list");
        }
        UM_CUDA_CHECK(cudaStreamWaitEvent(cs, copy_ev[act.arg], 0));
        waited[act.arg] = 1;
      } else if (act.kind == UM_ACT_WAIT_FLAG) {
        if ((rc = um_wait_geq(static_cast<const uint32_t*>(act.handle), (uint32_t)act.arg, cs))) {
          cleanup();
          return rc;
        }
      } else {
        cleanup();
        return fail(UM_EVALUE, "um_execute: unknown action kind " + std::to_string(act.kind));
      }
    }
    // join every pull (and the get stream) back into the compute stream
    for (int i = 0; i < P.ncopies; ++i)
      if (!waited[i]) UM_CUDA_CHECK(cudaStreamWaitEvent(cs, copy_ev[i], 0));
    cudaEvent_t gdone, done;
    if ((rc = event_on(gs, P.device, &gdone))) {
      cleanup();
      return rc;
    }
    events.push_back(gdone);
    UM_CUDA_CHECK(cudaStreamWaitEvent(cs, gdone, 0));
    if ((rc = event_on(cs, P.device, &done))) {
      cleanup();
      return rc;
    }
    events.push_back(done);
    rank_done.push_back(done);
    dev_done[P.device].push_back(done);
  }
  // replica reduction after the run-level barrier (runtime.py:376-386)
  for (int i = 0; i < nreduce; ++i) {
    const um_reduce_step& R = reduces[i];
    DeviceGuard g(R.device);
    auto it = st.reduce_streams.find(R.device);
    cudaStream_t rs;
    if (it == st.reduce_streams.end()) {
      UM_CUDA_CHECK(cudaStreamCreateWithFlags(&rs, cudaStreamNonBlocking));
      st.reduce_streams[R.device] = rs;
    } else {
      rs = it->second;
    }
    for (auto& kv : start) UM_CUDA_CHECK(cudaStreamWaitEvent(rs, kv.second, 0));
    for (cudaEvent_t e : rank_done) UM_CUDA_CHECK(cudaStreamWaitEvent(rs, e, 0));
    if ((rc = um_reduce_replicas(&R.dst, R.srcs, R.nsrc, R.mode, rs))) {
      cleanup();
      return rc;
    }
    cudaEvent_t done;
    if ((rc = event_on(rs, R.device, &done))) {
      cleanup();
      return rc;
    }
    events.push_back(done);
    dev_done[R.device].push_back(done);
  }
  // new per-device tails: one event that follows everything this call issued on the device
  for (auto& kv : dev_done) {
    const int dev = kv.first;
    DeviceGuard g(dev);
    cudaStream_t js;
    if ((rc = stream_for(st.rank_streams, -1 - dev, 2, dev, &js))) {   // per-device join stream
      cleanup();
      return rc;
    }
    for (cudaEvent_t e : kv.second) UM_CUDA_CHECK(cudaStreamWaitEvent(js, e, 0));
    cudaEvent_t tail;
    if ((rc = event_on(js, dev, &tail))) {
      cleanup();
      return rc;
    }
    auto old = st.tail.find(dev);
    if (old != st.tail.end()) cudaEventDestroy(old->second);
    st.tail[dev] = tail;
  }
  cleanup();
  return UM_OK;
}

extern "C" int um_execute_wait(void* stream, int32_t device) {
  // make a caller's stream (e.g. torch's current stream) wait for everything
  // um_execute issued on `device`
  Streams& st = S();
  std::lock_guard<std::mutex> lk(st.mu);
  auto it = st.tail.find(device);
  if (it == st.tail.end()) return UM_OK;
  DeviceGuard g(device);
  UM_CUDA_CHECK(cudaStreamWaitEvent(reinterpret_cast<cudaStream_t>(stream), it->second, 0));
  return UM_OK;
}

extern "C" int um_execute_after(void* stream, int32_t device) {
  // make the next um_execute on `device` start after the work queued on a caller's stream
  Streams& st = S();
  std::lock_guard<std::mutex> lk(st.mu);
  DeviceGuard g(device);
  cudaEvent_t e;
  UM_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  UM_CUDA_CHECK(cudaEventRecord(e, reinterpret_cast<cudaStream_t>(stream)));
  auto it = st.tail.find(device);
  if (it != st.tail.end()) {
    // keep both orders: join the old tail and the caller's stream on the device's join stream
    cudaStream_t js;
    int rc = stream_for(st.rank_streams, -1 - device, 2, device, &js);
    if (rc) return rc;
    UM_CUDA_CHECK(cudaStreamWaitEvent(js, it->second, 0));
    UM_CUDA_CHECK(cudaStreamWaitEvent(js, e, 0));
    cudaEventDestroy(e);
    cudaEventDestroy(it->second);
    UM_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    UM_CUDA_CHECK(cudaEventRecord(e, js));
  }
  st.tail[device] = e;
  return UM_OK;
}

extern "C" int um_sync_all(void) {
  // the run-level host barrier: every stream um_execute used has drained
  Streams& st = S();
  std::lock_guard<std::mutex> lk(st.mu);
  for (auto& kv : st.tail) {
    DeviceGuard g(kv.first);
    UM_CUDA_CHECK(cudaEventSynchronize(kv.second));
  }
  return UM_OK;
}

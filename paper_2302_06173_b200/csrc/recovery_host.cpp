// C++ recovery host over NCCL (recovery.cpp is absent from the
// reference): the consistency resolver's exchange, apply_undo and
// replica recovery, the ordered merge of parallel recovery, and NCCL-native
// failure detection / communicator repair.  This is
// the integrator-facing orchestration a C++ training system links instead of
// the Python/torch.distributed driver (recovery.py): plain pointers, one
// ncclComm_t per rw_comm, every transfer on a communicator stream ordered
// after the caller's stream.
//
// Conventions shared with the rest of the C ABI: status 0 = OK, 1 + Err for
// the reference's errors, RW_CUDA_ERROR / RW_INVALID_ARGUMENT otherwise; the
// thread-local message via rw_last_error_message().  NCCL failures map to
// RW_CHANNEL_BROKEN (errors.hpp ChannelBroken: "the detection signal").
#include <cuda_runtime.h>
#include <fcntl.h>
#include <nccl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <time.h>
#include <unistd.h>

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "internal.h"

namespace {

int hfail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  rwb::set_error(buf);
  return code;
}

#define HCUDA(call)                                                                          \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess) return hfail(RW_CUDA_ERROR, "CUDA error in %s: %s", #call,        \
                                        cudaGetErrorString(e_));                             \
  } while (0)

using Clock = std::chrono::steady_clock;

double ms_since(Clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

}  // namespace

// ------------------------------------------------------------------ rw_comm
struct rw_comm {
  ncclComm_t comm = nullptr;
  bool owned = false;
  int rank = 0;
  int size = 1;
  int device = 0;
  cudaStream_t stream = nullptr;  // the communicator's own stream
  // failure detection (rw_comm_watch)
  std::thread watcher;
  std::atomic<bool> stop{false};
  std::atomic<int> failed{0};      // RW_FAIL_* reason, 0 = healthy
  std::atomic<int> nccl_error{0};  // ncclResult_t seen by the poller
  uint32_t poll_us = 0;
  uint32_t timeout_ms = 0;
  std::mutex mu;                   // guards `inflight`
  std::deque<std::pair<cudaEvent_t, Clock::time_point>> inflight;  // watchdog: enqueued collectives
  std::vector<cudaEvent_t> free_events;
  Clock::time_point failed_at{};
  double detect_ms = -1.0;         // enqueue of the oldest stuck op -> detection
  // small exchange buffers (pinned host + device): a pageable copy would block
  // the host thread behind a collective that waits on a dead peer
  uint64_t* h_buf = nullptr;
  uint64_t* d_buf = nullptr;
  size_t buf_words = 0;
  // copy-engine chain (RW_RECOVER_CHAIN): peers' allocations mapped through
  // CUDA IPC once and kept (keyed by handle), the epoch counters the
  // predecessor writes, and the epoch of the current call
  std::vector<std::pair<std::array<uint8_t, 64>, void*>> ipc_maps;
  uint64_t* chain_ctr = nullptr;
  size_t chain_ctr_n = 0;
  uint64_t chain_epoch = 0;
};

namespace {

// Nonblocking communicators return ncclInProgress from enqueue / group calls;
// wait for completion of the host-side part (not the kernels) while watching
// the failure flag, so a dead peer can never wedge the host thread.
int nccl_settle(rw_comm* c, ncclResult_t r, const char* what) {
  // a host-side operation still in progress long after the watch timeout (or
  // 120 s unwatched) is a failure too: it waits on a peer that is gone.  The
  // host side of a fresh communicator's first collectives includes NCCL's lazy
  // connection setup (seconds on some boxes), so it gets at least 30 s; a dead
  // peer during a collective's device phase is the watchdog's job
  // (timeout_ms, measured per tracked batch).
  const auto t0 = Clock::now();
  const double limit = c->timeout_ms ? std::max(double(c->timeout_ms), 30000.0) : 120000.0;
  while (r == ncclInProgress) {
    if (c->failed.load()) return hfail(RW_CHANNEL_BROKEN, "ChannelBroken: %s: communicator failed", what);
    ncclResult_t a = ncclSuccess;
    if (ncclCommGetAsyncError(c->comm, &a) != ncclSuccess) break;
    r = a;
    if (r == ncclInProgress) {
      if (ms_since(t0) > limit) {
        c->detect_ms = ms_since(t0);
        c->failed = RW_COMM_FAILED_TIMEOUT;
        return hfail(RW_CHANNEL_BROKEN, "ChannelBroken: %s: no progress for %.0f ms", what, c->detect_ms);
      }
      std::this_thread::yield();
    }
  }
  if (r != ncclSuccess)
    return hfail(RW_CHANNEL_BROKEN, "ChannelBroken: %s: %s (%s)", what, ncclGetErrorString(r),
                 c->comm ? ncclGetLastError(c->comm) : "");
  return RW_OK;
}

#define HNCCL(c, call)                                \
  do {                                                \
    int s_ = nccl_settle((c), (call), #call);         \
    if (s_) return s_;                                \
  } while (0)

// Wait for the communicator stream without ever blocking on a collective
// that waits for a dead peer: poll, and give up once the watchdog has declared
// the communicator failed (its kernels are then terminated by the shrink /
// abort that repairs it).
int sync_comm(rw_comm* c, const char* what) {
  // unwatched communicators get the same bound as nccl_settle: no completion
  // in 120 s means a collective waits on a peer that is gone
  const auto t0 = Clock::now();
  for (;;) {
    const cudaError_t e = cudaStreamQuery(c->stream);
    if (e == cudaSuccess) break;
    if (e != cudaErrorNotReady) return hfail(RW_CUDA_ERROR, "CUDA error in %s: %s", what, cudaGetErrorString(e));
    if (c->failed.load()) return hfail(RW_CHANNEL_BROKEN, "ChannelBroken: %s: peer failure detected", what);
    if (!c->poll_us && ms_since(t0) > 120000.0) {
      c->detect_ms = ms_since(t0);
      c->failed = RW_COMM_FAILED_TIMEOUT;
      return hfail(RW_CHANNEL_BROKEN, "ChannelBroken: %s: no completion for %.0f ms", what, c->detect_ms);
    }
    std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
  if (c->failed.load()) return hfail(RW_CHANNEL_BROKEN, "ChannelBroken: %s: peer failure detected", what);
  return RW_OK;
}

// the watchdog tracks every batch of collectives the host issues
int track(rw_comm* c) {
  if (!c->poll_us) return RW_OK;
  cudaEvent_t ev = nullptr;
  {
    std::lock_guard<std::mutex> lk(c->mu);
    if (!c->free_events.empty()) {
      ev = c->free_events.back();
      c->free_events.pop_back();
    }
  }
  if (!ev) HCUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  HCUDA(cudaEventRecord(ev, c->stream));
  std::lock_guard<std::mutex> lk(c->mu);
  c->inflight.emplace_back(ev, Clock::now());
  return RW_OK;
}

// caller's stream -> comm stream ordering and back
int order_after(cudaStream_t waiter, cudaStream_t producer) {
  if (waiter == producer) return RW_OK;
  cudaEvent_t ev;
  HCUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  HCUDA(cudaEventRecord(ev, producer));
  HCUDA(cudaStreamWaitEvent(waiter, ev, 0));
  cudaEventDestroy(ev);
  return RW_OK;
}

int setup_comm(rw_comm* c) {
  int n = 0, r = 0, d = 0;
  if (ncclCommCount(c->comm, &n) != ncclSuccess || ncclCommUserRank(c->comm, &r) != ncclSuccess ||
      ncclCommCuDevice(c->comm, &d) != ncclSuccess)
    return hfail(RW_CHANNEL_BROKEN, "ChannelBroken: cannot query the NCCL communicator");
  c->size = n;
  c->rank = r;
  c->device = d;
  rwb::DeviceScope ds(d);
  HCUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  return RW_OK;
}

size_t elem_bytes(int dtype) { return dtype == RW_F64 ? 8 : 4; }

int ensure_bufs(rw_comm* c, size_t words) {
  if (words <= c->buf_words) return RW_OK;
  cudaFreeHost(c->h_buf);
  cudaFree(c->d_buf);
  c->h_buf = nullptr;
  c->d_buf = nullptr;
  c->buf_words = 0;
  words = std::max<size_t>(words, 64);
  HCUDA(cudaMallocHost(reinterpret_cast<void**>(&c->h_buf), words * 8));
  HCUDA(cudaMalloc(reinterpret_cast<void**>(&c->d_buf), words * 8));
  c->buf_words = words;
  return RW_OK;
}

void free_chain(rw_comm* c) {
  for (auto& m : c->ipc_maps) rw_ipc_close(m.second);
  c->ipc_maps.clear();
  if (c->chain_ctr) cudaFree(c->chain_ctr);
  c->chain_ctr = nullptr;
  c->chain_ctr_n = 0;
}

void free_bufs(rw_comm* c) {
  if (c->h_buf) cudaFreeHost(c->h_buf);
  if (c->d_buf) cudaFree(c->d_buf);
  c->h_buf = nullptr;
  c->d_buf = nullptr;
  c->buf_words = 0;
}

}  // namespace

// markers (and LAMB trust stacks) travel with the state: one broadcast from
// the root once its undo has finished, written into every other rank's state
static int replicate_meta(rw_comm* c, rw_state* s, const rw_hyper* h, int32_t root, std::vector<rw_group>& mk,
                          void* stream) {
  const uint32_t G = static_cast<uint32_t>(mk.size());
  const bool is_root = c->rank == root;
  auto cs = static_cast<cudaStream_t>(stream);
  int st = RW_OK;
  const int depth = RW_LAMB_TRUST_DEPTH;
  const bool lamb = h->kind == RW_LAMB;
  const size_t words = size_t(G) * 2 + (lamb ? size_t(G) * (depth + 1) : 0);
  std::vector<uint64_t> meta(words ? words : 1);
  if (is_root) {
    HCUDA(cudaStreamSynchronize(cs));  // the undo's markers are final
    if (G && (st = rw_state_read_groups(s, mk.data(), stream))) return st;
    for (uint32_t i = 0; i < G; ++i) meta[2 * i] = mk[i].t, meta[2 * i + 1] = mk[i].updated;
    if (lamb)
      for (uint32_t i = 0; i < G; ++i) {
        double vals[RW_LAMB_TRUST_DEPTH];
        uint32_t cnt = 0;
        if ((st = rw_state_saved_scalars(s, i, vals, depth, &cnt, stream))) return st;
        uint64_t* row = meta.data() + 2 * G + size_t(i) * (depth + 1);
        row[0] = cnt;
        std::memcpy(row + 1, vals, sizeof(double) * cnt);
      }
  }
  if (words) {
    if ((st = ensure_bufs(c, words))) return st;
    std::memcpy(c->h_buf, meta.data(), words * 8);
    HCUDA(cudaMemcpyAsync(c->d_buf, c->h_buf, words * 8, cudaMemcpyHostToDevice, c->stream));
    HNCCL(c, ncclBroadcast(c->d_buf, c->d_buf, words, ncclUint64, root, c->comm, c->stream));
    if ((st = track(c))) return st;
    HCUDA(cudaMemcpyAsync(c->h_buf, c->d_buf, words * 8, cudaMemcpyDeviceToHost, c->stream));
  }
  if ((st = sync_comm(c, "recover_replication"))) return st;
  if (words) std::memcpy(meta.data(), c->h_buf, words * 8);
  if (!is_root) {
    for (uint32_t i = 0; i < G; ++i) mk[i].t = meta[2 * i], mk[i].updated = static_cast<uint32_t>(meta[2 * i + 1]);
    if (G && (st = rw_state_write_groups(s, mk.data(), stream))) return st;
    if (lamb)
      for (uint32_t i = 0; i < G; ++i) {
        const uint64_t* row = meta.data() + 2 * G + size_t(i) * (depth + 1);
        double vals[RW_LAMB_TRUST_DEPTH];
        std::memcpy(vals, row + 1, sizeof(vals));
        if ((st = rw_state_set_saved_scalars(s, i, vals, static_cast<uint32_t>(row[0]), stream))) return st;
      }
  }
  return RW_OK;
}

// apply_undo + recover_replication over the copy engines, as a chain
// (recovery.recover_replication_chain): ranks in the order root, then the
// others ascending; every rank but the last maps its successor's buffers and
// epoch counters through CUDA IPC (handles exchanged with one ncclAllGather);
// the root undoes run i on the caller's stream while the communicator stream
// copies run i-1 into the successor's HBM (cudaMemcpyAsync over NVLink, no
// kernel) and bumps the successor's counter for that run; every other rank's
// communicator stream waits for its own counter and forwards the run.
static int chain_transfer(rw_comm* c, rw_state* s, const rw_hyper* h, int32_t root, const uint8_t* actions,
                          bool undo, const std::vector<rw_group>& mk, uint64_t total, size_t es,
                          const std::vector<void*>& bufs, const std::vector<std::pair<uint32_t, uint32_t>>& runs,
                          cudaStream_t cs, uint64_t* bytes_out) {
  const int n = c->size, nb = static_cast<int>(bufs.size());
  const uint32_t G = static_cast<uint32_t>(mk.size());
  const size_t npieces = runs.size();
  if (c->chain_ctr_n < npieces) {  // counters persist across calls; epochs only grow
    if (c->chain_ctr) cudaFree(c->chain_ctr);
    HCUDA(cudaMalloc(&c->chain_ctr, std::max<size_t>(npieces, 16) * 8));
    HCUDA(cudaMemset(c->chain_ctr, 0, std::max<size_t>(npieces, 16) * 8));
    c->chain_ctr_n = std::max<size_t>(npieces, 16);
    c->chain_epoch = 0;
  }
  uint64_t* counters = c->chain_ctr;
  // every rank reallocates together (same npieces), so the epochs stay in step
  const uint64_t epoch = ++c->chain_epoch;
  // exchange: per rank nb + 1 records of (64-byte handle, 8-byte offset) = 9 words each
  const size_t rec = 9, per = (nb + 1) * rec;
  int st = ensure_bufs(c, per * n);
  if (st) return st;
  std::vector<uint64_t> mine(per, 0);
  for (int b = 0; b <= nb; ++b) {
    void* p = b < nb ? bufs[b] : static_cast<void*>(counters);
    if ((st = rw_ipc_export(p, mine.data() + b * rec, &mine[b * rec + 8]))) return st;
  }
  std::memcpy(c->h_buf, mine.data(), per * 8);
  HCUDA(cudaMemcpyAsync(c->d_buf + per * c->rank, c->h_buf, per * 8, cudaMemcpyHostToDevice, c->stream));
  HNCCL(c, ncclAllGather(c->d_buf + per * c->rank, c->d_buf, per, ncclUint64, c->comm, c->stream));
  if ((st = track(c))) return st;
  HCUDA(cudaMemcpyAsync(c->h_buf, c->d_buf, per * n * 8, cudaMemcpyDeviceToHost, c->stream));
  if ((st = sync_comm(c, "recover_replication (chain handles)"))) return st;
  std::vector<int> chain{root};
  for (int r = 0; r < n; ++r)
    if (r != root) chain.push_back(r);
  const int pos = static_cast<int>(std::find(chain.begin(), chain.end(), c->rank) - chain.begin());
  const int next = pos + 1 < n ? chain[pos + 1] : -1;
  std::vector<char*> dst(nb + 1, nullptr);
  if (next >= 0) {
    const uint64_t* rec0 = c->h_buf + per * next;
    for (int b = 0; b <= nb; ++b) {
      std::array<uint8_t, 64> key;
      std::memcpy(key.data(), rec0 + b * rec, 64);
      void* base = nullptr;
      for (auto& m : c->ipc_maps)
        if (m.first == key) base = m.second;
      if (!base) {  // map each allocation of the successor once per communicator
        if ((st = rw_ipc_import(key.data(), &base))) return st;
        c->ipc_maps.emplace_back(key, base);
      }
      dst[b] = static_cast<char*>(base) + rec0[b * rec + 8];
    }
  }
  cudaEvent_t ev;
  HCUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  constexpr size_t kLead = 2;
  std::vector<cudaEvent_t> copied(npieces, nullptr);
  for (auto& e : copied) HCUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  uint64_t bytes = 0;
  for (size_t k = 0; k < npieces; ++k) {
    const uint32_t g0 = runs[k].first, g1 = runs[k].second;
    const uint64_t lo = g0 == 0 ? 0 : mk[g0].offset, hi = g1 < G ? mk[g1].offset : total;
    if (pos == 0) {
      if (undo) {
        std::vector<uint32_t> ids;
        for (uint32_t i = g0; i < g1; ++i)
          if (actions[i] == RW_ACT_UNDO) ids.push_back(i);
        // pace the undo two runs ahead of the copies: a burst of every run's
        // undo at full HBM bandwidth would starve the copy engines' reads
        if (!ids.empty() && k >= kLead) HCUDA(cudaStreamWaitEvent(cs, copied[k - kLead], 0));
        if (!ids.empty() && (st = rw_optimizer_undo(s, h, ids.data(), static_cast<uint32_t>(ids.size()), cs)))
          return st;
      }
      HCUDA(cudaEventRecord(ev, cs));
      HCUDA(cudaStreamWaitEvent(c->stream, ev, 0));
    } else if ((st = rw_stream_wait_u64(c->stream, counters + k, epoch))) {  // the predecessor's copy landed
      return st;
    }
    if (next >= 0) {
      std::vector<void*> d(nb);
      std::vector<const void*> src(nb);
      std::vector<uint64_t> len(nb, (hi - lo) * es);
      for (int b = 0; b < nb; ++b) {
        d[b] = dst[b] + lo * es;
        src[b] = static_cast<const char*>(bufs[b]) + lo * es;
      }
      if ((st = rw_copy_async(d.data(), src.data(), len.data(), static_cast<uint32_t>(nb), c->stream))) return st;
      if ((st = rw_stream_write_u64(c->stream, reinterpret_cast<uint64_t*>(dst[nb]) + k, epoch))) return st;
      if (pos == 0) HCUDA(cudaEventRecord(copied[k], c->stream));
    }
    bytes += (hi - lo) * es * nb;
  }
  cudaEventDestroy(ev);
  for (auto& e : copied) cudaEventDestroy(e);
  // every hop has landed everywhere before anyone moves on (the next call may
  // overwrite the same buffers)
  HNCCL(c, ncclAllReduce(c->d_buf, c->d_buf, 1, ncclUint64, ncclMax, c->comm, c->stream));
  if ((st = track(c))) return st;
  *bytes_out = bytes;
  return RW_OK;
}

extern "C" {

int rw_nccl_unique_id(void* id_out) {
  if (!id_out) return hfail(RW_INVALID_ARGUMENT, "null argument");
  ncclUniqueId id;
  const ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return hfail(RW_CHANNEL_BROKEN, "ncclGetUniqueId: %s", ncclGetErrorString(r));
  std::memcpy(id_out, &id, sizeof(id));
  return RW_OK;
}

int rw_comm_init(rw_comm** out, const void* unique_id, int32_t nranks, int32_t rank, int32_t device) {
  if (!out || !unique_id || nranks < 1 || rank < 0 || rank >= nranks)
    return hfail(RW_INVALID_ARGUMENT, "bad communicator arguments");
  rwb::DeviceScope ds(device);
  HCUDA(cudaSetDevice(device));
  auto* c = new rw_comm();
  c->owned = true;
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof(id));
  ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
  cfg.blocking = 0;  // nonblocking: a dead peer cannot wedge the host (abort / shrink stay possible)
  ncclResult_t r = ncclCommInitRankConfig(&c->comm, nranks, id, rank, &cfg);
  int st = nccl_settle(c, r, "ncclCommInitRankConfig");
  if (!st) st = setup_comm(c);
  if (st) {
    if (c->comm) ncclCommAbort(c->comm);
    delete c;
    return st;
  }
  *out = c;
  return RW_OK;
}

int rw_comm_from_nccl(rw_comm** out, void* nccl_comm) {
  if (!out || !nccl_comm) return hfail(RW_INVALID_ARGUMENT, "null argument");
  auto* c = new rw_comm();
  c->comm = static_cast<ncclComm_t>(nccl_comm);
  c->owned = false;
  int st = setup_comm(c);
  if (st) {
    delete c;
    return st;
  }
  *out = c;
  return RW_OK;
}

int32_t rw_comm_rank(const rw_comm* c) { return c ? c->rank : -1; }
int32_t rw_comm_size(const rw_comm* c) { return c ? c->size : 0; }
void* rw_comm_stream(rw_comm* c) { return c ? c->stream : nullptr; }
void* rw_comm_nccl(rw_comm* c) { return c ? c->comm : nullptr; }

static void stop_watch(rw_comm* c) {
  c->stop = true;
  if (c->watcher.joinable()) c->watcher.join();
  std::lock_guard<std::mutex> lk(c->mu);
  for (auto& p : c->inflight) cudaEventDestroy(p.first);
  for (auto e : c->free_events) cudaEventDestroy(e);
  c->inflight.clear();
  c->free_events.clear();
}

int rw_comm_destroy(rw_comm* c) {
  if (!c) return RW_OK;
  rwb::DeviceScope ds(c->device);
  stop_watch(c);
  int st = RW_OK;
  if (c->owned && c->comm) {
    if (c->failed.load()) {
      ncclCommAbort(c->comm);
    } else {
      ncclResult_t r = ncclCommFinalize(c->comm);
      st = nccl_settle(c, r, "ncclCommFinalize");
      if (st) ncclCommAbort(c->comm);
      else ncclCommDestroy(c->comm);
    }
  }
  if (c->stream) cudaStreamDestroy(c->stream);
  free_chain(c);
  free_bufs(c);
  delete c;
  return st;
}

int rw_comm_abort(rw_comm* c) {
  if (!c) return RW_OK;
  rwb::DeviceScope ds(c->device);
  stop_watch(c);
  if (c->comm) ncclCommAbort(c->comm);
  c->comm = nullptr;
  if (c->stream) cudaStreamDestroy(c->stream);
  free_chain(c);
  free_bufs(c);
  delete c;
  return RW_OK;
}

// ---- failure detection (poll ncclCommGetAsyncError) ----
int rw_comm_watch(rw_comm* c, uint32_t poll_us, uint32_t timeout_ms) {
  if (!c || !poll_us) return hfail(RW_INVALID_ARGUMENT, "bad watch arguments");
  if (c->watcher.joinable()) return RW_OK;
  c->poll_us = poll_us;
  c->timeout_ms = timeout_ms;
  c->stop = false;
  c->watcher = std::thread([c] {
    cudaSetDevice(c->device);
    while (!c->stop.load()) {
      ncclResult_t a = ncclSuccess;
      if (c->comm && ncclCommGetAsyncError(c->comm, &a) == ncclSuccess && a != ncclSuccess && a != ncclInProgress) {
        c->nccl_error = static_cast<int>(a);
        c->failed_at = Clock::now();
        c->detect_ms = 0.0;
        c->failed = RW_COMM_FAILED_NCCL_ERROR;
        return;
      }
      {
        std::lock_guard<std::mutex> lk(c->mu);
        while (!c->inflight.empty() && cudaEventQuery(c->inflight.front().first) == cudaSuccess) {
          c->free_events.push_back(c->inflight.front().first);
          c->inflight.pop_front();
        }
        if (c->timeout_ms && !c->inflight.empty()) {
          const double waited = ms_since(c->inflight.front().second);
          if (waited > c->timeout_ms) {  // a collective has not completed: a peer is gone (fail-stop)
            c->failed_at = Clock::now();
            c->detect_ms = waited;
            c->failed = RW_COMM_FAILED_TIMEOUT;
            return;
          }
        }
      }
      std::this_thread::sleep_for(std::chrono::microseconds(c->poll_us));
    }
  });
  return RW_OK;
}

int rw_comm_failed(rw_comm* c, int32_t* reason, double* detect_ms) {
  if (!c) return hfail(RW_INVALID_ARGUMENT, "null communicator");
  if (reason) *reason = c->failed.load();
  if (detect_ms) *detect_ms = c->detect_ms;
  return RW_OK;
}

int rw_comm_shrink(rw_comm* c, const int32_t* exclude, int32_t n_exclude, rw_comm** out) {
  if (!c || !out || (n_exclude && !exclude)) return hfail(RW_INVALID_ARGUMENT, "null argument");
  rwb::DeviceScope ds(c->device);
  stop_watch(c);  // the parent is being torn down: its in-flight work is abandoned
  auto* nc = new rw_comm();
  nc->owned = true;
  std::vector<int> ex(exclude, exclude + n_exclude);
  // NCCL_SHRINK_ABORT: terminate the parent's outstanding operations (they
  // wait on the dead rank) before shrinking; the child inherits the parent's
  // (nonblocking) configuration
  const int flags = c->failed.load() ? NCCL_SHRINK_ABORT : NCCL_SHRINK_DEFAULT;
  ncclResult_t r = ncclCommShrink(c->comm, ex.data(), n_exclude, &nc->comm, nullptr, flags);
  int st = RW_OK;
  if (r != ncclSuccess && r != ncclInProgress) {
    st = hfail(RW_CHANNEL_BROKEN, "ChannelBroken: ncclCommShrink: %s", ncclGetErrorString(r));
  } else {
    // nonblocking: the child handle and its state settle asynchronously
    const auto t0 = Clock::now();
    for (;;) {
      if (nc->comm) {
        ncclResult_t a = ncclInProgress;
        if (ncclCommGetAsyncError(nc->comm, &a) != ncclSuccess) a = ncclInternalError;
        if (a == ncclSuccess) break;
        if (a != ncclInProgress) {
          st = hfail(RW_CHANNEL_BROKEN, "ChannelBroken: ncclCommShrink child: %s", ncclGetErrorString(a));
          break;
        }
      } else {
        ncclResult_t a = ncclSuccess;
        ncclCommGetAsyncError(c->comm, &a);
        if (a != ncclSuccess && a != ncclInProgress && ms_since(t0) > 1000.0) {
          st = hfail(RW_CHANNEL_BROKEN, "ChannelBroken: ncclCommShrink: parent %s, no child",
                     ncclGetErrorString(a));
          break;
        }
      }
      if (ms_since(t0) > 30000.0) {
        st = hfail(RW_CHANNEL_BROKEN, "ChannelBroken: ncclCommShrink did not complete (result %d, flags %d, child %p)",
                   int(r), flags, static_cast<void*>(nc->comm));
        break;
      }
      std::this_thread::sleep_for(std::chrono::microseconds(100));
    }
  }
  if (!st) st = setup_comm(nc);
  if (st) {
    if (nc->comm) ncclCommAbort(nc->comm);
    delete nc;
    return st;
  }
  *out = nc;
  return RW_OK;
}

// ---- heartbeat membership (the "global key-value store" of SPEC:253-261, node-local) ----
// Each slot holds its rank's last beat as CLOCK_MONOTONIC nanoseconds (one
// clock for every process of the node), so any observer can tell how long a
// rank has been silent without having watched it beat.
namespace {
uint64_t mono_ns() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return uint64_t(ts.tv_sec) * 1000000000ull + uint64_t(ts.tv_nsec);
}
}  // namespace

struct rw_membership {
  int fd = -1;
  uint64_t* slots = nullptr;  // [nranks] last-beat timestamps in a shared file
  int32_t rank = 0, nranks = 0;
  std::thread beat;
  std::atomic<bool> stop{false};
};

int rw_membership_open(rw_membership** out, const char* path, int32_t rank, int32_t nranks, uint32_t beat_us) {
  if (!out || !path || nranks < 1 || rank < -1 || rank >= nranks || !beat_us)
    return hfail(RW_INVALID_ARGUMENT, "bad membership arguments");
  const int fd = ::open(path, O_RDWR | O_CREAT, 0644);
  if (fd < 0) return hfail(RW_STORAGE_ERROR, "StorageError: cannot open %s", path);
  const size_t bytes = sizeof(uint64_t) * size_t(nranks);
  struct stat sb;
  if (fstat(fd, &sb) != 0 || (static_cast<size_t>(sb.st_size) < bytes && ftruncate(fd, bytes) != 0)) {
    ::close(fd);
    return hfail(RW_STORAGE_ERROR, "StorageError: cannot size %s", path);
  }
  void* p = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  if (p == MAP_FAILED) {
    ::close(fd);
    return hfail(RW_STORAGE_ERROR, "StorageError: cannot map %s", path);
  }
  auto* m = new rw_membership();
  m->fd = fd;
  m->slots = static_cast<uint64_t*>(p);
  m->rank = rank;
  m->nranks = nranks;
  if (rank >= 0) {  // rank -1: observer only
    __atomic_store_n(&m->slots[rank], mono_ns(), __ATOMIC_RELEASE);
    m->beat = std::thread([m, beat_us] {
      while (!m->stop.load()) {
        __atomic_store_n(&m->slots[m->rank], mono_ns(), __ATOMIC_RELEASE);
        std::this_thread::sleep_for(std::chrono::microseconds(beat_us));
      }
    });
  }
  *out = m;
  return RW_OK;
}

// ranks silent for more than timeout_ms (fail-stop: a process that died stops
// beating; a slot never written counts as silent), ascending
int rw_membership_dead(rw_membership* m, uint32_t timeout_ms, int32_t* dead, int32_t cap, int32_t* n_dead) {
  if (!m || !n_dead || (cap && !dead)) return hfail(RW_INVALID_ARGUMENT, "null argument");
  int n = 0;
  const uint64_t now = mono_ns(), lim = uint64_t(timeout_ms) * 1000000ull;
  for (int r = 0; r < m->nranks; ++r) {
    if (r == m->rank) continue;
    const uint64_t v = __atomic_load_n(&m->slots[r], __ATOMIC_ACQUIRE);
    if (now > v && now - v > lim) {
      if (n < cap) dead[n] = r;
      ++n;
    }
  }
  *n_dead = n;
  return RW_OK;
}

int rw_membership_close(rw_membership* m) {
  if (!m) return RW_OK;
  m->stop = true;
  if (m->beat.joinable()) m->beat.join();
  munmap(m->slots, sizeof(uint64_t) * size_t(m->nranks));
  ::close(m->fd);
  delete m;
  return RW_OK;
}

// ---- resolver exchange (consensus = MIN over survivors) ----
int rw_resolve(rw_state* s, const rw_hyper* h, rw_comm* c, int32_t policy, const uint8_t* grad_ready,
               uint8_t* actions, rw_resolution* out, void* stream) {
  if (!h || !c || !out) return hfail(RW_INVALID_ARGUMENT, "null argument");
  rwb::DeviceScope ds(c->device);
  const uint32_t n = s ? rw_state_num_groups(s) : 0;
  if (n && !actions) return hfail(RW_INVALID_ARGUMENT, "actions buffer needed for a state");
  std::vector<rw_group> mk(n);
  if (n) {
    int st = rw_state_read_groups(s, mk.data(), stream);
    if (st) return st;
  }
  rw_resolve_summary loc{};
  int st = rw_resolve_summarize(mk.data(), n, grad_ready, h, UINT64_MAX, &loc);
  if (st) return st;
  // exchange 1: (t_min MIN, t_max MAX); exchange 2: costs / blocks (MAX)
  if ((st = ensure_bufs(c, 8))) return st;
  uint64_t* d = c->d_buf;
  uint64_t* hv = c->h_buf;
  hv[0] = loc.t_min;
  hv[1] = loc.t_max;
  HCUDA(cudaMemcpyAsync(d, hv, 2 * sizeof(uint64_t), cudaMemcpyHostToDevice, c->stream));
  HNCCL(c, ncclGroupStart());
  HNCCL(c, ncclAllReduce(d, d, 1, ncclUint64, ncclMin, c->comm, c->stream));
  HNCCL(c, ncclAllReduce(d + 1, d + 1, 1, ncclUint64, ncclMax, c->comm, c->stream));
  HNCCL(c, ncclGroupEnd());
  if (int t = track(c)) return t;
  HCUDA(cudaMemcpyAsync(hv, d, 2 * sizeof(uint64_t), cudaMemcpyDeviceToHost, c->stream));
  if ((st = sync_comm(c, "resolve"))) return st;
  const uint64_t lo = hv[0], hi = hv[1];
  rw_resolve_summary s2{};
  st = rw_resolve_summarize(mk.data(), n, grad_ready, h, lo, &s2);
  if (st) return st;
  hv[2] = s2.undo_elems;
  hv[3] = s2.redo_elems;
  hv[4] = s2.redo_blocked;
  hv[5] = s2.undo_blocked;
  HCUDA(cudaMemcpyAsync(d + 2, hv + 2, 4 * sizeof(uint64_t), cudaMemcpyHostToDevice, c->stream));
  HNCCL(c, ncclAllReduce(d + 2, d + 2, 4, ncclUint64, ncclMax, c->comm, c->stream));
  if (int t = track(c)) return t;
  HCUDA(cudaMemcpyAsync(hv + 2, d + 2, 4 * sizeof(uint64_t), cudaMemcpyDeviceToHost, c->stream));
  if ((st = sync_comm(c, "resolve"))) return st;
  const uint64_t costs[4] = {hv[2], hv[3], hv[4], hv[5]};
  rw_resolve_summary glob{};
  glob.t_min = lo;
  glob.t_max = hi;
  glob.undo_elems = costs[0];
  glob.redo_elems = costs[1];
  glob.redo_blocked = costs[2];
  glob.undo_blocked = costs[3];
  uint64_t target = 0;
  int32_t strategy = 0;
  std::vector<uint8_t> acts(n);
  st = rw_resolve_plan(&glob, policy, mk.data(), n, acts.data(), &target, &strategy);
  if (st) return st;
  out->strategy = strategy;
  out->target = target;
  out->t_min = lo;
  out->t_max = hi;
  out->n_undo = out->n_redo = 0;
  for (uint32_t i = 0; i < n; ++i) {
    actions[i] = acts[i];
    out->n_undo += acts[i] == RW_ACT_UNDO;
    out->n_redo += acts[i] == RW_ACT_REDO;
  }
  return RW_OK;
}

// ---- apply_undo / redo ----
int rw_apply_resolution(rw_state* s, const rw_hyper* h, const uint8_t* actions, int32_t strategy, const void* grad,
                        void* stream) {
  if (!s || !h || !actions) return hfail(RW_INVALID_ARGUMENT, "null argument");
  if (strategy == RW_STRATEGY_GLOBAL_ROLLBACK)
    return hfail(RW_NOT_INVERTIBLE, "NotInvertible: the plan requires a global checkpoint rollback (SPEC:488)");
  const uint32_t n = rw_state_num_groups(s);
  std::vector<uint32_t> ids;
  if (strategy == RW_STRATEGY_UNDO) {
    // decide on t (SURVEY §8a a13 spec gap): re-arm flags cleared at iteration end
    std::vector<rw_group> mk(n);
    int st = rw_state_read_groups(s, mk.data(), stream);
    if (st) return st;
    bool rearm = false;
    for (uint32_t i = 0; i < n; ++i)
      if (actions[i] == RW_ACT_UNDO && !mk[i].updated) mk[i].updated = 1, rearm = true;
    if (rearm && (st = rw_state_write_groups(s, mk.data(), stream))) return st;
    // undo in reverse update order: update order = reverse layer order, so ascending group index
    for (uint32_t i = 0; i < n; ++i)
      if (actions[i] == RW_ACT_UNDO) ids.push_back(i);
    return ids.empty() ? RW_OK : rw_optimizer_undo(s, h, ids.data(), static_cast<uint32_t>(ids.size()), stream);
  }
  if (strategy == RW_STRATEGY_REDO) {
    if (!grad) return hfail(RW_INVALID_ARGUMENT, "redo needs the synchronised gradient buffer");
    for (uint32_t i = n; i-- > 0;)  // update order (reverse layer order)
      if (actions[i] == RW_ACT_REDO) ids.push_back(i);
    return ids.empty() ? RW_OK
                       : rw_optimizer_step(s, h, ids.data(), static_cast<uint32_t>(ids.size()), grad, UINT32_MAX,
                                           stream);
  }
  return RW_OK;
}

// ---- recover_replication ----
int rw_recover_replication(rw_state* s, const rw_hyper* h, rw_comm* c, int32_t root, const uint8_t* actions,
                           int32_t strategy, uint32_t flags, uint32_t pieces, void* stream, uint64_t* bytes_out) {
  if (!s || !h || !c) return hfail(RW_INVALID_ARGUMENT, "null argument");
  if (root < 0 || root >= c->size) return hfail(RW_NO_REPLICA, "NoReplica: root rank %d out of range", root);
  rwb::DeviceScope ds(c->device);
  const uint32_t G = rw_state_num_groups(s);
  const bool is_root = c->rank == root;
  if (is_root && G && !actions) return hfail(RW_INVALID_ARGUMENT, "the survivor needs its actions");
  int32_t dtype = 0;
  uint64_t total = 0;
  int32_t dev = 0;
  int st = rw_state_info(s, &dtype, &total, &dev);
  if (st) return st;
  const size_t es = elem_bytes(dtype);
  std::vector<rw_group> mk(G);
  if (G && (st = rw_state_read_groups(s, mk.data(), stream))) return st;
  if (is_root && strategy == RW_STRATEGY_REDO) return hfail(RW_INVALID_ARGUMENT, "apply a redo before replicating");
  if (is_root && strategy == RW_STRATEGY_GLOBAL_ROLLBACK)
    return hfail(RW_NOT_INVERTIBLE, "NotInvertible: the plan requires a global checkpoint rollback (SPEC:488)");
  const bool undo = is_root && strategy == RW_STRATEGY_UNDO;
  if (undo) {  // re-arm (decide on t), as rw_apply_resolution
    bool rearm = false;
    for (uint32_t i = 0; i < G; ++i)
      if (actions[i] == RW_ACT_UNDO && !mk[i].updated) mk[i].updated = 1, rearm = true;
    if (rearm && (st = rw_state_write_groups(s, mk.data(), stream))) return st;
  }
  std::vector<void*> bufs;
  for (int w : {0, 1, 2, 3}) {
    if (w == 1 && !(flags & RW_RECOVER_INCLUDE_GRAD)) continue;
    if (void* p = rw_state_ptr(s, w)) bufs.push_back(p);
  }
  // contiguous runs of whole groups, ~total/pieces elements each (same on every rank)
  if (pieces == 0) pieces = 16;
  std::vector<std::pair<uint32_t, uint32_t>> runs;
  {
    uint64_t acc = 0, tot = 0;
    for (auto& g : mk) tot += g.len;
    uint32_t start = 0;
    for (uint32_t i = 0; i < G; ++i) {
      acc += mk[i].len;
      if (double(acc) >= double(tot) * double(runs.size() + 1) / pieces || i + 1 == G) {
        runs.emplace_back(start, i + 1);
        start = i + 1;
      }
    }
  }
  auto cs = static_cast<cudaStream_t>(stream);
  if ((st = order_after(c->stream, cs))) return st;
  if (flags & RW_RECOVER_CHAIN) {
    uint64_t bytes = 0;
    if ((st = chain_transfer(c, s, h, root, actions, undo, mk, total, es, bufs, runs, cs, &bytes))) return st;
    if ((st = replicate_meta(c, s, h, root, mk, stream))) return st;
    if ((st = order_after(cs, c->stream))) return st;
    if (bytes_out) *bytes_out = bytes;
    return RW_OK;
  }
  cudaEvent_t ev;
  HCUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  uint64_t bytes = 0;
  for (auto [g0, g1] : runs) {
    // runs tile the whole buffer (alignment padding included), so replicas end byte-identical
    const uint64_t lo = g0 == 0 ? 0 : mk[g0].offset, hi = g1 < G ? mk[g1].offset : total;
    if (undo) {  // undo this run on the caller's stream, then broadcast it from the comm stream
      std::vector<uint32_t> ids;
      for (uint32_t i = g0; i < g1; ++i)
        if (actions[i] == RW_ACT_UNDO) ids.push_back(i);
      if (!ids.empty() && (st = rw_optimizer_undo(s, h, ids.data(), static_cast<uint32_t>(ids.size()), stream))) {
        cudaEventDestroy(ev);
        return st;
      }
      HCUDA(cudaEventRecord(ev, cs));
      HCUDA(cudaStreamWaitEvent(c->stream, ev, 0));
    }
    HNCCL(c, ncclGroupStart());
    for (void* b : bufs)
      HNCCL(c, ncclBroadcast(static_cast<char*>(b) + lo * es, static_cast<char*>(b) + lo * es, (hi - lo) * es,
                             ncclUint8, root, c->comm, c->stream));
    HNCCL(c, ncclGroupEnd());
    if ((st = track(c))) return st;
    bytes += (hi - lo) * es * bufs.size();
  }
  cudaEventDestroy(ev);
  if ((st = replicate_meta(c, s, h, root, mk, stream))) return st;
  if ((st = order_after(cs, c->stream))) return st;
  if (bytes_out) *bytes_out = bytes;
  return RW_OK;
}

// ---- ordered merge of parallel recovery ----
// Shard j of the flat gradient ([j*chunk, (j+1)*chunk) clipped to n, chunk a
// multiple of 64 elements) is owned by rank j.  Every rank sends shard j of
// each micro-batch partial it computed (mb mod d == rank) to rank j; rank j
// sums ITS shard over mb = 0..m-1 in ascending order (ordered_sum, bit-identical
// to the sequential replay) and the shards are all-gathered into `out`.
uint64_t rw_ordered_reduce_chunk(uint64_t n, int32_t nranks) {
  if (nranks < 1) return 0;
  const uint64_t per = (n + uint64_t(nranks) - 1) / uint64_t(nranks);
  return (per + 63) / 64 * 64;
}

uint64_t rw_ordered_reduce_scratch_elems(uint64_t n, uint32_t m, int32_t nranks, int32_t rank) {
  if (nranks < 1 || rank < 0 || rank >= nranks) return 0;
  uint32_t foreign = 0;
  for (uint32_t mb = 0; mb < m; ++mb) foreign += (int32_t(mb % uint32_t(nranks)) != rank);
  return uint64_t(foreign) * rw_ordered_reduce_chunk(n, nranks);
}

int rw_ordered_reduce(rw_comm* c, const float* const* parts, uint32_t m, uint64_t n, float* out, float* scratch,
                      uint64_t scratch_elems, void* stream) {
  if (!c || !parts || !out || m == 0) return hfail(RW_INVALID_ARGUMENT, "bad ordered_reduce arguments");
  rwb::DeviceScope ds(c->device);
  const int d = c->size, me = c->rank;
  const uint64_t chunk = rw_ordered_reduce_chunk(n, d);
  if (scratch_elems < rw_ordered_reduce_scratch_elems(n, m, d, me) || (!scratch && scratch_elems))
    return hfail(RW_INVALID_ARGUMENT, "scratch too small (rw_ordered_reduce_scratch_elems)");
  auto lo_of = [&](int j) { return std::min<uint64_t>(n, uint64_t(j) * chunk); };
  auto hi_of = [&](int j) { return std::min<uint64_t>(n, uint64_t(j + 1) * chunk); };
  for (uint32_t mb = 0; mb < m; ++mb)
    if (int32_t(mb % uint32_t(d)) == me && !parts[mb]) return hfail(RW_MISSING_LOG_DATA, "MissingLogData: partial of mb %u", mb);
  auto cs = static_cast<cudaStream_t>(stream);
  int st = order_after(c->stream, cs);
  if (st) return st;
  // 1) point-to-point: my partials' shards out, the other owners' partials of my shard in
  std::vector<const void*> mine(m, nullptr);
  const uint64_t mlo = lo_of(me), mhi = hi_of(me);
  uint64_t slot = 0;
  HNCCL(c, ncclGroupStart());
  for (uint32_t mb = 0; mb < m; ++mb) {
    const int owner = int(mb % uint32_t(d));
    if (owner == me) {
      for (int j = 0; j < d; ++j)
        if (j != me && hi_of(j) > lo_of(j))
          HNCCL(c, ncclSend(parts[mb] + lo_of(j), hi_of(j) - lo_of(j), ncclFloat, j, c->comm, c->stream));
      mine[mb] = parts[mb] + mlo;
    } else {
      float* dst = scratch + slot * chunk;
      ++slot;
      if (mhi > mlo) HNCCL(c, ncclRecv(dst, mhi - mlo, ncclFloat, owner, c->comm, c->stream));
      mine[mb] = dst;
    }
  }
  HNCCL(c, ncclGroupEnd());
  if ((st = track(c))) return st;
  // 2) ascending-mb ordered sum of my shard, in place in `out`
  if (mhi > mlo) {
    const int e = rwb::launch_ordered_sum(RW_F32, mine.data(), m, mhi - mlo, out + mlo, c->stream);
    if (e) return hfail(RW_CUDA_ERROR, "ordered_sum: %s", cudaGetErrorString(static_cast<cudaError_t>(e)));
  }
  // 3) all-gather of the shards (in place: rank j's shard already sits at j*chunk)
  // out holds chunk * d elements (rw_ordered_reduce_out_elems); the tail past n is padding
  HNCCL(c, ncclAllGather(out + uint64_t(me) * chunk, out, chunk, ncclFloat, c->comm, c->stream));
  if ((st = track(c))) return st;
  return order_after(cs, c->stream);
}

uint64_t rw_ordered_reduce_out_elems(uint64_t n, int32_t nranks) {
  return rw_ordered_reduce_chunk(n, nranks) * uint64_t(nranks < 1 ? 1 : nranks);
}

}  // extern "C"

// Logging capture path (logstore.cpp is absent from the
// reference): upstream-backup logging of boundary tensors off the critical
// path, in native code.
//
//   producer (training thread)          committer (std::thread)
//   ---------------------------         ------------------------------
//   event on producer stream            wait entry event (copy done)
//   copy stream waits that event        append record to chunk file
//   CRC32 kernel  -> d_crc[slot]        every chunk_records: close,
//   D2H payload   -> pinned slab          rename .tmp -> final (atomic)
//   D2H crc       -> h_crc[slot]        release slab bytes, advance
//   event; push SPSC entry              committed watermark
//
// The committer hands completed records round-robin to `lanes` writer
// threads; each lane owns its current chunk file (records stay whole and in
// order within a file; a record's position in the log is its (iteration,
// micro-batch, direction) key, not its file).  One thread's write() into the
// page cache tops out at ~3.4 GB/s and writers sharing a file serialise on
// its inode lock, so separate files are what lets capture scale.  Slab bytes
// are released in record order as the lanes finish.
//
// The training stream is never blocked; the host producer blocks only when
// the pinned slab or the queue is full (backpressure), which bounds memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "internal.h"

namespace {
int lfail(int code, const std::string& msg) {
  rwb::set_error(msg.c_str());
  return code;
}
#define LCUDA(call)                                                                              \
  do {                                                                                           \
    cudaError_t e_ = (call);                                                                     \
    if (e_ != cudaSuccess) return lfail(RW_CUDA_ERROR, std::string("CUDA error in " #call ": ") + \
                                                           cudaGetErrorString(e_));              \
  } while (0)

constexpr uint32_t kQ = 1024;  // queue entries in flight
constexpr uint16_t kVersion = 1;

size_t elem_bytes(uint32_t dtype) { return dtype == RW_F64 ? 8 : dtype == RW_BF16 ? 2 : 4; }

struct Entry {
  rw_log_record rec;
  uint64_t off = 0;      // slab offset (absolute, monotonic)
  uint64_t end = 0;      // slab offset after this record (incl. wrap padding)
  uint32_t slot = 0;
  cudaEvent_t ev = nullptr;
};

void put_u16(std::vector<uint8_t>& b, uint16_t v) {
  b.push_back(uint8_t(v));
  b.push_back(uint8_t(v >> 8));
}
void put_u32(std::vector<uint8_t>& b, uint32_t v) {
  for (int i = 0; i < 4; ++i) b.push_back(uint8_t(v >> (8 * i)));
}
void put_u64(std::vector<uint8_t>& b, uint64_t v) {
  for (int i = 0; i < 8; ++i) b.push_back(uint8_t(v >> (8 * i)));
}
}  // namespace

struct rw_logger {
  std::string dir;
  uint32_t machine = 0;
  uint32_t chunk_records = 64;
  int device = 0;
  uint8_t* slab = nullptr;
  uint64_t slab_size = 0;
  uint64_t slab_head = 0;               // producer-owned
  std::atomic<uint64_t> slab_tail{0};   // committer releases
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t prod_ev = nullptr;
  uint32_t* d_crc = nullptr;            // kQ slots
  uint32_t* h_crc = nullptr;            // pinned, kQ slots
  uint32_t* d_scratch = nullptr;
  uint64_t scratch_words = 0;
  Entry ring[kQ];
  std::atomic<uint64_t> q_head{0}, q_tail{0};
  std::thread th;
  std::atomic<bool> stop{false};
  std::atomic<bool> finalize_req{false};
  std::mutex mu;
  std::condition_variable cv;
  std::atomic<uint64_t> committed{0};
  std::atomic<int> err{0};
  std::string errmsg;
  // writer lanes: each owns its current chunk file
  struct Lane {
    struct Job {
      rw_log_record rec;
      const uint8_t* payload;
      std::atomic<int>* done;
    };
    std::thread th;
    std::mutex mu;
    std::condition_variable cv;
    std::deque<Job> q;
    bool close_req = false, stop = false;
    FILE* cur = nullptr;
    uint32_t in_chunk = 0;
    std::string cur_tmp, cur_final;
  };
  std::vector<std::unique_ptr<Lane>> lanes;
  std::atomic<uint64_t> seq{0};  // chunk file numbers, shared by the lanes
  uint64_t dispatched = 0;
  struct InFlight {
    uint64_t end;
    std::unique_ptr<std::atomic<int>> done;
  };
  std::deque<InFlight> inflight;  // committer-owned, record order
};

namespace {

bool open_chunk(rw_logger* L, rw_logger::Lane* W) {
  char name[64];
  std::snprintf(name, sizeof(name), "m%04u_%08llu.swft", L->machine,
                static_cast<unsigned long long>(L->seq.fetch_add(1)));
  W->cur_final = L->dir + "/" + name;
  W->cur_tmp = W->cur_final + ".tmp";
  W->cur = std::fopen(W->cur_tmp.c_str(), "wb");
  if (!W->cur) return false;
  std::vector<uint8_t> h = {'S', 'W', 'F', 'T'};
  put_u16(h, kVersion);
  put_u32(h, L->machine);
  return std::fwrite(h.data(), 1, h.size(), W->cur) == h.size();
}

bool close_chunk(rw_logger::Lane* W) {
  if (!W->cur) return true;
  bool ok = std::fflush(W->cur) == 0;
  ok &= std::fclose(W->cur) == 0;
  W->cur = nullptr;
  ok &= std::rename(W->cur_tmp.c_str(), W->cur_final.c_str()) == 0;  // atomic commit
  W->in_chunk = 0;
  return ok;
}

bool write_record(rw_logger* L, rw_logger::Lane* W, const rw_log_record& r, const uint8_t* payload) {
  if (!W->cur && !open_chunk(L, W)) return false;
  std::vector<uint8_t> h;
  // record_len = bytes after this field (ids 24 + flags 4 + shape + payload_len 8 + payload + crc 4);
  // its low 32 bits only — the u64 payload_len below is authoritative.
  const uint32_t len = 4 + 4 + 8 + 4 + 4 + 8 * r.ndim + 8 + 4;
  put_u32(h, len + static_cast<uint32_t>(r.payload_bytes & 0xFFFFFFFFu));
  put_u32(h, r.sender);
  put_u32(h, r.receiver);
  put_u64(h, r.iteration);
  put_u32(h, r.mb);
  h.push_back(uint8_t(r.direction));
  h.push_back(uint8_t(r.dtype));
  h.push_back(uint8_t(r.ndim));
  h.push_back(0);
  for (uint32_t i = 0; i < r.ndim; ++i) put_u64(h, r.shape[i]);
  put_u64(h, r.payload_bytes);
  if (std::fwrite(h.data(), 1, h.size(), W->cur) != h.size()) return false;
  if (r.payload_bytes && std::fwrite(payload, 1, r.payload_bytes, W->cur) != r.payload_bytes) return false;
  std::vector<uint8_t> c;
  put_u32(c, r.crc32);
  if (std::fwrite(c.data(), 1, 4, W->cur) != 4) return false;
  if (++W->in_chunk >= L->chunk_records) return close_chunk(W);
  return true;
}

void lane_main(rw_logger* L, rw_logger::Lane* W) {
  while (true) {
    rw_logger::Lane::Job j{};
    bool have = false, do_close = false;
    {
      std::unique_lock<std::mutex> lk(W->mu);
      W->cv.wait(lk, [&] { return W->stop || W->close_req || !W->q.empty(); });
      if (!W->q.empty()) {
        j = W->q.front();
        W->q.pop_front();
        have = true;
      } else if (W->close_req) {
        do_close = true;
      } else {
        return;  // stop, drained
      }
    }
    if (have) {
      if (!L->err && !write_record(L, W, j.rec, j.payload)) {
        L->errmsg = "StorageError: short write in " + L->dir;
        L->err = RW_STORAGE_ERROR;
      }
      j.done->store(1, std::memory_order_release);
    } else if (do_close) {
      if (!close_chunk(W) && !L->err) {
        L->errmsg = "StorageError: cannot commit log chunk in " + L->dir;
        L->err = RW_STORAGE_ERROR;
      }
      std::lock_guard<std::mutex> lk(W->mu);
      W->close_req = false;
    }
    L->cv.notify_all();
  }
}

// release slab bytes of finished records, in record order; wait_all drains
void retire(rw_logger* L, bool wait_all) {
  while (!L->inflight.empty()) {
    auto& f = L->inflight.front();
    if (!f.done->load(std::memory_order_acquire)) {
      if (!wait_all) return;
      std::unique_lock<std::mutex> lk(L->mu);
      L->cv.wait_for(lk, std::chrono::microseconds(200));
      continue;
    }
    L->slab_tail.store(f.end, std::memory_order_release);
    L->committed.fetch_add(1);
    L->inflight.pop_front();
    L->cv.notify_all();
  }
}

// every lane closes (commits) its partial chunk
bool close_all(rw_logger* L) {
  retire(L, true);
  for (auto& W : L->lanes) {
    std::lock_guard<std::mutex> lk(W->mu);
    W->close_req = true;
    W->cv.notify_all();
  }
  for (auto& W : L->lanes) {
    while (true) {
      {
        std::lock_guard<std::mutex> lk(W->mu);
        if (!W->close_req) break;
      }
      std::unique_lock<std::mutex> lk(L->mu);
      L->cv.wait_for(lk, std::chrono::microseconds(200));
    }
  }
  return !L->err;
}

void committer(rw_logger* L) {
  cudaSetDevice(L->device);
  while (true) {
    uint64_t tail = L->q_tail.load(std::memory_order_relaxed);
    if (tail == L->q_head.load(std::memory_order_acquire)) {
      if (L->finalize_req.load()) {
        close_all(L);
        L->finalize_req = false;
        L->cv.notify_all();
        continue;
      }
      if (L->stop.load()) break;
      retire(L, false);
      std::unique_lock<std::mutex> lk(L->mu);
      L->cv.wait_for(lk, std::chrono::milliseconds(1));
      continue;
    }
    Entry& e = L->ring[tail % kQ];
    cudaError_t ce = cudaEventSynchronize(e.ev);
    if (ce != cudaSuccess && !L->err) {
      L->errmsg = std::string("CUDA error in log copy: ") + cudaGetErrorString(ce);
      L->err = RW_CUDA_ERROR;
    }
    e.rec.crc32 = L->h_crc[e.slot];
    const uint8_t* payload = L->slab + (e.off % L->slab_size);
    rw_logger::InFlight f{e.end, std::make_unique<std::atomic<int>>(0)};
    std::atomic<int>* done = f.done.get();
    L->inflight.push_back(std::move(f));
    rw_logger::Lane* W = L->lanes[L->dispatched++ % L->lanes.size()].get();
    {
      std::lock_guard<std::mutex> lk(W->mu);
      W->q.push_back(rw_logger::Lane::Job{e.rec, payload, done});
    }
    W->cv.notify_all();
    L->q_tail.store(tail + 1, std::memory_order_release);
    retire(L, false);
    L->cv.notify_all();
  }
}

}  // namespace

extern "C" {

int rw_crc32_device(const void* data, uint64_t n, uint32_t* out_dev, void* stream) {
  rwb::DeviceScope dev_scope(rwb::DeviceScope::device_of(data));
  if ((!data && n) || !out_dev) return lfail(RW_INVALID_ARGUMENT, "null argument");
  // the scratch comes from the device's default stream-ordered pool; keep a
  // few MB of it cached (release threshold) so a call does not map and unmap
  // memory each time (the default threshold of 0 returns it at every sync)
  static rwb::DeviceOnce pool_once;
  pool_once.run([](int dev) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = 64ull << 20;
      uint64_t cur = 0;
      if (cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &cur) == cudaSuccess && cur < keep)
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    return 0;  // best effort: the threshold only saves remapping
  });
  uint32_t* scratch = nullptr;
  LCUDA(cudaMallocAsync(reinterpret_cast<void**>(&scratch), rwb::crc32_scratch_words(n) * 4,
                        static_cast<cudaStream_t>(stream)));
  int e = rwb::launch_crc32(data, n, out_dev, scratch, stream);
  cudaFreeAsync(scratch, static_cast<cudaStream_t>(stream));
  if (e) return lfail(RW_CUDA_ERROR, std::string("crc32 kernel: ") + cudaGetErrorString(cudaError_t(e)));
  return RW_OK;
}

int rw_logger_create(rw_logger** out, const char* dir, uint32_t machine, uint32_t chunk_records,
                     uint64_t pinned_bytes, int32_t device) {
  if (!out || !dir || chunk_records == 0 || pinned_bytes < 4096) return lfail(RW_INVALID_ARGUMENT, "bad argument");
  *out = nullptr;
  if (rw_device_count() == 0) return lfail(RW_CUDA_ERROR, "no CUDA device visible: the B200 path has no CPU fallback");
  auto* L = new rw_logger();
  L->dir = dir;
  L->machine = machine;
  L->chunk_records = chunk_records;
  L->device = device;
  L->slab_size = pinned_bytes;
  auto bail = [&](int code) {
    rw_logger_destroy(L);
    return code;
  };
  if (cudaSetDevice(device) != cudaSuccess) return bail(lfail(RW_CUDA_ERROR, "cudaSetDevice failed"));
  if (cudaMallocHost(&L->slab, pinned_bytes) != cudaSuccess) return bail(lfail(RW_CUDA_ERROR, "pinned slab allocation"));
  if (cudaStreamCreateWithFlags(&L->copy_stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&L->prod_ev, cudaEventDisableTiming) != cudaSuccess ||
      cudaMalloc(&L->d_crc, kQ * 4) != cudaSuccess || cudaMallocHost(&L->h_crc, kQ * 4) != cudaSuccess)
    return bail(lfail(RW_CUDA_ERROR, "logger CUDA resources"));
  for (auto& e : L->ring)
    if (cudaEventCreateWithFlags(&e.ev, cudaEventDisableTiming) != cudaSuccess)
      return bail(lfail(RW_CUDA_ERROR, "logger events"));
  // probe the directory
  std::string probe = L->dir + "/.probe";
  FILE* f = std::fopen(probe.c_str(), "wb");
  if (!f) return bail(lfail(RW_STORAGE_ERROR, "StorageError: cannot write to " + L->dir));
  std::fclose(f);
  std::remove(probe.c_str());
  // one writer lane per host core, 4..16 (page-cache writes scale with threads:
  // 16 lanes capture 19-21 GB/s vs 16-19 with 8 on a 16-core box,
  // profiles/r02/logging_slab_lanes.log)
  int nl = int(std::min(16u, std::max(4u, std::thread::hardware_concurrency())));
  if (const char* ev = std::getenv("RW_LOG_LANES")) nl = std::max(1, std::atoi(ev));
  for (int i = 0; i < nl; ++i) {
    L->lanes.emplace_back(new rw_logger::Lane());
    L->lanes.back()->th = std::thread(lane_main, L, L->lanes.back().get());
  }
  L->th = std::thread(committer, L);
  *out = L;
  return RW_OK;
}

int rw_logger_log(rw_logger* L, const rw_log_record* rec, const void* dev_payload, void* producer_stream) {
  rwb::DeviceScope dev_scope(rwb::DeviceScope::device_of(dev_payload));
  if (!L || !rec || (!dev_payload && rec->payload_bytes)) return lfail(RW_INVALID_ARGUMENT, "null argument");
  if (rec->ndim > 4) return lfail(RW_INVALID_SHAPE, "InvalidShape: ndim > 4");
  if (L->err) return lfail(L->err, L->errmsg);
  uint64_t elems = 1;
  for (uint32_t i = 0; i < rec->ndim; ++i) elems *= rec->shape[i];
  const uint64_t bytes = rec->payload_bytes;
  if (rec->ndim && elems * elem_bytes(rec->dtype) != bytes)
    return lfail(RW_SHAPE_MISMATCH, "ShapeMismatch: payload bytes do not match shape x dtype");
  if (bytes > L->slab_size) return lfail(RW_TOO_LARGE, "TooLarge: record larger than the pinned slab");
  LCUDA(cudaSetDevice(L->device));
  // queue space (backpressure)
  while (L->q_head.load() - L->q_tail.load(std::memory_order_acquire) >= kQ) {
    std::unique_lock<std::mutex> lk(L->mu);
    L->cv.wait_for(lk, std::chrono::milliseconds(1));
  }
  // contiguous slab range; skip to the next wrap if the record would straddle it
  uint64_t off = L->slab_head;
  const uint64_t in_slab = off % L->slab_size;
  if (in_slab + bytes > L->slab_size) off += L->slab_size - in_slab;
  const uint64_t end = off + ((bytes + 255) & ~uint64_t(255));
  while (end - L->slab_tail.load(std::memory_order_acquire) > L->slab_size) {
    if (L->err) return lfail(L->err, L->errmsg);
    std::unique_lock<std::mutex> lk(L->mu);
    L->cv.wait_for(lk, std::chrono::milliseconds(1));
  }
  L->slab_head = end;
  const uint64_t h = L->q_head.load();
  Entry& e = L->ring[h % kQ];
  e.rec = *rec;
  e.rec.crc32 = 0;
  e.off = off;
  e.end = end;
  e.slot = static_cast<uint32_t>(h % kQ);
  auto ps = static_cast<cudaStream_t>(producer_stream);
  LCUDA(cudaEventRecord(L->prod_ev, ps));
  LCUDA(cudaStreamWaitEvent(L->copy_stream, L->prod_ev, 0));
  const uint64_t need = rwb::crc32_scratch_words(bytes);
  if (need > L->scratch_words) {
    LCUDA(cudaStreamSynchronize(L->copy_stream));
    cudaFree(L->d_scratch);
    L->d_scratch = nullptr;
    LCUDA(cudaMalloc(&L->d_scratch, need * 4));
    L->scratch_words = need;
  }
  int ke = rwb::launch_crc32(dev_payload, bytes, L->d_crc + e.slot, L->d_scratch, L->copy_stream);
  if (ke) return lfail(RW_CUDA_ERROR, std::string("crc32 kernel: ") + cudaGetErrorString(cudaError_t(ke)));
  if (bytes)
    LCUDA(cudaMemcpyAsync(L->slab + (off % L->slab_size), dev_payload, bytes, cudaMemcpyDeviceToHost, L->copy_stream));
  LCUDA(cudaMemcpyAsync(L->h_crc + e.slot, L->d_crc + e.slot, 4, cudaMemcpyDeviceToHost, L->copy_stream));
  LCUDA(cudaEventRecord(e.ev, L->copy_stream));
  L->q_head.store(h + 1, std::memory_order_release);
  L->cv.notify_all();
  return RW_OK;
}

int rw_logger_flush(rw_logger* L, uint64_t* committed) {
  if (!L) return lfail(RW_INVALID_ARGUMENT, "null logger");
  while (L->q_tail.load(std::memory_order_acquire) != L->q_head.load()) {
    std::unique_lock<std::mutex> lk(L->mu);
    L->cv.wait_for(lk, std::chrono::milliseconds(1));
  }
  L->finalize_req = true;
  L->cv.notify_all();
  while (L->finalize_req.load()) {
    std::unique_lock<std::mutex> lk(L->mu);
    L->cv.wait_for(lk, std::chrono::milliseconds(1));
  }
  if (committed) *committed = L->committed.load();
  if (L->err) return lfail(L->err, L->errmsg);
  return RW_OK;
}

void* rw_logger_stream(rw_logger* L) { return L ? static_cast<void*>(L->copy_stream) : nullptr; }

int rw_logger_destroy(rw_logger* L) {
  if (!L) return RW_OK;
  int st = RW_OK;
  if (L->th.joinable()) {
    st = rw_logger_flush(L, nullptr);
    L->stop = true;
    L->cv.notify_all();
    L->th.join();
  }
  for (auto& W : L->lanes) {
    {
      std::lock_guard<std::mutex> lk(W->mu);
      W->stop = true;
    }
    W->cv.notify_all();
    if (W->th.joinable()) W->th.join();
  }
  if (L->copy_stream) cudaStreamSynchronize(L->copy_stream);
  for (auto& e : L->ring)
    if (e.ev) cudaEventDestroy(e.ev);
  if (L->prod_ev) cudaEventDestroy(L->prod_ev);
  if (L->copy_stream) cudaStreamDestroy(L->copy_stream);
  cudaFree(L->d_crc);
  cudaFree(L->d_scratch);
  cudaFreeHost(L->h_crc);
  cudaFreeHost(L->slab);
  delete L;
  return st;
}

}  // extern "C"

// ---------------- reader ----------------
struct rw_log_reader {
  FILE* f = nullptr;
  uint32_t machine = 0;
};

namespace {
bool rd(FILE* f, void* p, size_t n) { return std::fread(p, 1, n, f) == n; }
template <class T>
bool rd_le(FILE* f, T* v) {
  uint8_t b[sizeof(T)];
  if (!rd(f, b, sizeof(T))) return false;
  T r = 0;
  for (size_t i = 0; i < sizeof(T); ++i) r |= T(b[i]) << (8 * i);
  *v = r;
  return true;
}
}  // namespace

extern "C" {

int rw_log_open(rw_log_reader** out, const char* path, uint32_t* machine) {
  if (!out || !path) return lfail(RW_INVALID_ARGUMENT, "null argument");
  *out = nullptr;
  FILE* f = std::fopen(path, "rb");
  if (!f) return lfail(RW_MISSING_LOG_DATA, std::string("MissingLogData: cannot open ") + path);
  char magic[4];
  uint16_t ver = 0;
  uint32_t m = 0;
  if (!rd(f, magic, 4) || std::memcmp(magic, "SWFT", 4) != 0 || !rd_le(f, &ver) || ver != kVersion ||
      !rd_le(f, &m)) {
    std::fclose(f);
    return lfail(RW_CORRUPT_LOG, std::string("CorruptLog: bad header in ") + path);
  }
  auto* r = new rw_log_reader();
  r->f = f;
  r->machine = m;
  if (machine) *machine = m;
  *out = r;
  return RW_OK;
}

int rw_log_next(rw_log_reader* r, rw_log_record* rec, void* payload, uint64_t cap, int32_t* eof) {
  if (!r || !rec || !eof) return lfail(RW_INVALID_ARGUMENT, "null argument");
  *eof = 0;
  uint32_t len = 0;
  uint8_t b0;
  if (std::fread(&b0, 1, 1, r->f) != 1) {
    *eof = 1;
    return RW_OK;
  }
  std::ungetc(b0, r->f);
  std::memset(rec, 0, sizeof(*rec));
  uint8_t dir = 0, dt = 0, nd = 0, pad = 0;
  if (!rd_le(r->f, &len) || !rd_le(r->f, &rec->sender) || !rd_le(r->f, &rec->receiver) ||
      !rd_le(r->f, &rec->iteration) || !rd_le(r->f, &rec->mb) || !rd(r->f, &dir, 1) || !rd(r->f, &dt, 1) ||
      !rd(r->f, &nd, 1) || !rd(r->f, &pad, 1) || nd > 4)
    return lfail(RW_CORRUPT_LOG, "CorruptLog: truncated record header");
  rec->direction = dir;
  rec->dtype = dt;
  rec->ndim = nd;
  for (uint32_t i = 0; i < nd; ++i)
    if (!rd_le(r->f, &rec->shape[i])) return lfail(RW_CORRUPT_LOG, "CorruptLog: truncated shape");
  if (!rd_le(r->f, &rec->payload_bytes)) return lfail(RW_CORRUPT_LOG, "CorruptLog: truncated length");
  const uint32_t expect = 4 + 4 + 8 + 4 + 4 + 8 * nd + 8 + 4 + static_cast<uint32_t>(rec->payload_bytes & 0xFFFFFFFFu);
  if (len != expect) return lfail(RW_CORRUPT_LOG, "CorruptLog: record length mismatch");
  if (rec->payload_bytes > cap) return lfail(RW_TOO_LARGE, "TooLarge: payload larger than the buffer");
  if (rec->payload_bytes && !rd(r->f, payload, rec->payload_bytes))
    return lfail(RW_CORRUPT_LOG, "CorruptLog: truncated payload");
  if (!rd_le(r->f, &rec->crc32)) return lfail(RW_CORRUPT_LOG, "CorruptLog: truncated checksum");
  return RW_OK;
}

int rw_log_skip(rw_log_reader* r, rw_log_record* rec, int32_t* eof) {
  if (!r || !rec || !eof) return lfail(RW_INVALID_ARGUMENT, "null argument");
  *eof = 0;
  uint8_t b0;
  if (std::fread(&b0, 1, 1, r->f) != 1) {
    *eof = 1;
    return RW_OK;
  }
  std::ungetc(b0, r->f);
  std::memset(rec, 0, sizeof(*rec));
  uint32_t len = 0;
  uint8_t dir = 0, dt = 0, nd = 0, pad = 0;
  if (!rd_le(r->f, &len) || !rd_le(r->f, &rec->sender) || !rd_le(r->f, &rec->receiver) ||
      !rd_le(r->f, &rec->iteration) || !rd_le(r->f, &rec->mb) || !rd(r->f, &dir, 1) || !rd(r->f, &dt, 1) ||
      !rd(r->f, &nd, 1) || !rd(r->f, &pad, 1) || nd > 4)
    return lfail(RW_CORRUPT_LOG, "CorruptLog: truncated record header");
  rec->direction = dir;
  rec->dtype = dt;
  rec->ndim = nd;
  for (uint32_t i = 0; i < nd; ++i)
    if (!rd_le(r->f, &rec->shape[i])) return lfail(RW_CORRUPT_LOG, "CorruptLog: truncated shape");
  if (!rd_le(r->f, &rec->payload_bytes)) return lfail(RW_CORRUPT_LOG, "CorruptLog: truncated length");
  if (std::fseek(r->f, static_cast<long>(rec->payload_bytes), SEEK_CUR) != 0 || !rd_le(r->f, &rec->crc32))
    return lfail(RW_CORRUPT_LOG, "CorruptLog: truncated payload");
  return RW_OK;
}

void rw_log_close(rw_log_reader* r) {
  if (!r) return;
  if (r->f) std::fclose(r->f);
  delete r;
}

}  // extern "C"

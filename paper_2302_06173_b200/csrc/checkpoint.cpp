// Global checkpoint store + log garbage collection (SPEC:389-392
// CheckpointManifest, SPEC:423-438 write_checkpoint / load_checkpoint /
// gc_logs; PAPER §3 "global checkpointing is performed periodically", §5.1
// "All earlier logging files are obsoleted after a global checkpointing").
// The reference has no source for these; wire.cpp:129-142
// gives its atomic-write idiom (write .tmp, rename), which is kept here.
//
// On-disk layout under `dir`:
//   ck_<iter:016>/w<worker:05>/<blob>.bin   raw bytes of a host buffer, or
//   ck_<iter:016>/w<worker:05>/<blob>.bin.<k>  part k of a device buffer
//   ck_<iter:016>/w<worker:05>.wm           worker manifest: names, sizes, CRC32s
//   MANIFEST_<iter:016>                     global commit marker
// Commit order: blobs written + fsync'd -> worker manifest (tmp, fsync,
// rename) -> every worker's manifest present -> MANIFEST (tmp, fsync, rename).
// Hence "manifest visible <=> all blobs fully written"; a crash anywhere
// before the final rename leaves the previous MANIFEST the latest valid one.
//
// Data path: device buffers move in 32 MiB chunks through 16 I/O workers,
// each with its own pinned chunk and copy stream (D2H + pwrite / pread +
// H2D at the chunk's file offset), so PCIe copies, page-cache copies and the
// storage work in parallel.  Each device blob's CRC32 (the wire.cpp polynomial) is
// computed on the GPU at HBM speed; load recomputes it on the GPU after the
// H2D and compares with the manifest.
#include <cuda_runtime.h>
#include <dirent.h>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cinttypes>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "internal.h"

namespace {

int cfail(int code, const std::string& msg) {
  rwb::set_error(msg.c_str());
  return code;
}
#define CCUDA(call)                                                                              \
  do {                                                                                           \
    cudaError_t e_ = (call);                                                                     \
    if (e_ != cudaSuccess) return cfail(RW_CUDA_ERROR, std::string("CUDA error in " #call ": ") + \
                                                           cudaGetErrorString(e_));              \
  } while (0)

constexpr uint64_t kChunk = 32ull << 20;  // pinned staging chunk per worker
#ifndef RW_CKPT_WORKERS
#define RW_CKPT_WORKERS 16  // = the GPU box's host cores: 27-29 / 30-32 GB/s write / load vs 19-21 / 22-23 with 8
#endif
constexpr int kWorkers = RW_CKPT_WORKERS;  // I/O threads, each with its own stream + buffer

// CRC32 (reflected 0xEDB88320), the wire.cpp:31-38 function, for host blobs
uint32_t crc32_host(const void* p, uint64_t n) {
  static uint32_t tab[256];
  static bool init = false;
  if (!init) {
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c & 1u) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
      tab[i] = c;
    }
    init = true;
  }
  uint32_t c = 0xFFFFFFFFu;
  const auto* b = static_cast<const uint8_t*>(p);
  for (uint64_t i = 0; i < n; ++i) c = tab[(c ^ b[i]) & 0xFFu] ^ (c >> 8);
  return c ^ 0xFFFFFFFFu;
}

// Staging pool shared by all calls (allocating pinned memory is slow): one
// pinned chunk + one copy stream per I/O worker.
struct Ring {
  std::mutex mu;
  void* buf[kWorkers] = {};
  cudaStream_t st[kWorkers] = {};
  cudaEvent_t start = nullptr;
  uint32_t* d_crc = nullptr;
  uint32_t* d_scratch = nullptr;
  uint64_t scratch_words = 0;
  int device = -1;
};
Ring g_ring;

int ring_ready(Ring& R) {
  int dev = 0;
  CCUDA(cudaGetDevice(&dev));
  if (R.device == dev && R.buf[0]) return RW_OK;
  if (R.buf[0]) {  // different device: rebuild on this one
    for (int i = 0; i < kWorkers; ++i) {
      cudaFreeHost(R.buf[i]);
      cudaStreamDestroy(R.st[i]);
      R.buf[i] = nullptr;
    }
    cudaEventDestroy(R.start);
    cudaFree(R.d_crc);
    cudaFree(R.d_scratch);
    R.d_crc = nullptr;
    R.d_scratch = nullptr;
    R.scratch_words = 0;
  }
  for (int i = 0; i < kWorkers; ++i) {
    CCUDA(cudaMallocHost(&R.buf[i], kChunk));
    CCUDA(cudaStreamCreateWithFlags(&R.st[i], cudaStreamNonBlocking));
  }
  CCUDA(cudaEventCreateWithFlags(&R.start, cudaEventDisableTiming));
  CCUDA(cudaMalloc(&R.d_crc, sizeof(uint32_t)));
  R.device = dev;
  return RW_OK;
}

// Move one device blob to (to_file) or from its part files: the blob's
// kChunk pieces are split into nparts contiguous parts, worker w moves part w
// (one async copy on its own stream + one pwrite/pread per chunk) into its own
// file, so the copies, the page cache and the storage run in parallel and no
// two writers share an inode lock.  Ordered after prior work on `cs`;
// complete (host-synchronised) on return.
uint32_t parts_for(uint64_t bytes) {
  const uint64_t nch = (bytes + kChunk - 1) / kChunk;
  return static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(kWorkers, nch)));
}
uint64_t part_chunks(uint64_t bytes, uint32_t nparts) {
  const uint64_t nch = (bytes + kChunk - 1) / kChunk;
  return (nch + nparts - 1) / nparts;
}
uint64_t part_bytes(uint64_t bytes, uint32_t nparts, uint32_t w) {
  const uint64_t per = part_chunks(bytes, nparts) * kChunk;
  const uint64_t lo = std::min<uint64_t>(bytes, w * per), hi = std::min<uint64_t>(bytes, (w + 1) * per);
  return hi - lo;
}
std::string part_path(const std::string& base, uint32_t w) { return base + "." + std::to_string(w); }

int staged_io(Ring& R, bool to_file, const std::vector<int>& fds, void* dev, uint64_t bytes, cudaStream_t cs,
              const std::string& path) {
  int device = 0;
  CCUDA(cudaGetDevice(&device));
  CCUDA(cudaEventRecord(R.start, cs));
  const uint32_t nparts = static_cast<uint32_t>(fds.size());
  const uint64_t nch = (bytes + kChunk - 1) / kChunk, per = part_chunks(bytes, nparts);
  std::vector<int> status(nparts, RW_OK);
  std::vector<std::string> errs(nparts);
  auto work = [&](uint32_t w) {
    if (cudaSetDevice(device) != cudaSuccess || cudaStreamWaitEvent(R.st[w], R.start, 0) != cudaSuccess) {
      status[w] = RW_CUDA_ERROR;
      errs[w] = "checkpoint worker setup failed";
      return;
    }
    const int fd = fds[w];
    for (uint64_t c = w * per; c < std::min<uint64_t>(nch, (w + 1) * per); ++c) {
      const uint64_t off = c * kChunk, len = std::min(kChunk, bytes - off), foff = off - w * per * kChunk;
      char* d = static_cast<char*>(dev) + off;
      if (to_file) {
        if (cudaMemcpyAsync(R.buf[w], d, len, cudaMemcpyDeviceToHost, R.st[w]) != cudaSuccess ||
            cudaStreamSynchronize(R.st[w]) != cudaSuccess) {
          status[w] = RW_CUDA_ERROR;
          errs[w] = "checkpoint D2H failed";
          return;
        }
        const char* p = static_cast<const char*>(R.buf[w]);
        uint64_t left = len, at = foff;
        while (left) {
          const ssize_t k = ::pwrite(fd, p, left, static_cast<off_t>(at));
          if (k < 0 && errno == EINTR) continue;
          if (k <= 0) {
            status[w] = RW_STORAGE_ERROR;
            errs[w] = "StorageError: short write on " + part_path(path, w);
            return;
          }
          p += k;
          at += uint64_t(k);
          left -= uint64_t(k);
        }
      } else {
        char* p = static_cast<char*>(R.buf[w]);
        uint64_t left = len, at = foff;
        while (left) {
          const ssize_t k = ::pread(fd, p, left, static_cast<off_t>(at));
          if (k < 0 && errno == EINTR) continue;
          if (k <= 0) {
            status[w] = RW_STORAGE_ERROR;
            errs[w] = "StorageError: short read on " + part_path(path, w);
            return;
          }
          p += k;
          at += uint64_t(k);
          left -= uint64_t(k);
        }
        if (cudaMemcpyAsync(d, R.buf[w], len, cudaMemcpyHostToDevice, R.st[w]) != cudaSuccess ||
            cudaStreamSynchronize(R.st[w]) != cudaSuccess) {
          status[w] = RW_CUDA_ERROR;
          errs[w] = "checkpoint H2D failed";
          return;
        }
      }
    }
    if (to_file && ::fsync(fd) != 0) {
      status[w] = RW_STORAGE_ERROR;
      errs[w] = "StorageError: fsync failed on " + part_path(path, w);
    }
  };
  std::vector<std::thread> th;
  for (uint32_t w = 1; w < nparts; ++w) th.emplace_back(work, w);
  work(0);
  for (auto& t : th) t.join();
  for (uint32_t w = 0; w < nparts; ++w)
    if (status[w]) return cfail(status[w], errs[w]);
  return RW_OK;
}

int device_crc(Ring& R, const void* dev, uint64_t n, cudaStream_t st, uint32_t* out) {
  const uint64_t need = rwb::crc32_scratch_words(n);
  if (need > R.scratch_words) {
    cudaFree(R.d_scratch);
    R.d_scratch = nullptr;
    CCUDA(cudaMalloc(&R.d_scratch, need * 4));
    R.scratch_words = need;
  }
  int e = rwb::launch_crc32(dev, n, R.d_crc, R.d_scratch, st);
  if (e) return cfail(RW_CUDA_ERROR, std::string("crc32 kernel: ") + cudaGetErrorString(cudaError_t(e)));
  CCUDA(cudaMemcpyAsync(out, R.d_crc, 4, cudaMemcpyDeviceToHost, st));
  CCUDA(cudaStreamSynchronize(st));
  return RW_OK;
}

std::string iter_dir(const std::string& dir, uint64_t it) {
  char b[64];
  std::snprintf(b, sizeof(b), "/ck_%016" PRIu64, it);
  return dir + b;
}
std::string worker_dir(const std::string& dir, uint64_t it, uint32_t w) {
  char b[32];
  std::snprintf(b, sizeof(b), "/w%05u", w);
  return iter_dir(dir, it) + b;
}
std::string manifest_path(const std::string& dir, uint64_t it) {
  char b[64];
  std::snprintf(b, sizeof(b), "/MANIFEST_%016" PRIu64, it);
  return dir + b;
}

bool valid_name(const char* s) {
  if (!s || !*s || std::strlen(s) > 200) return false;
  for (const char* p = s; *p; ++p)
    if (!(std::isalnum(static_cast<unsigned char>(*p)) || *p == '.' || *p == '_' || *p == '-')) return false;
  return true;
}

int mkdirs(const std::string& p) {
  std::string cur;
  for (size_t i = 0; i <= p.size(); ++i) {
    if (i == p.size() || p[i] == '/') {
      if (!cur.empty() && ::mkdir(cur.c_str(), 0755) != 0 && errno != EEXIST)
        return cfail(RW_STORAGE_ERROR, "StorageError: cannot create " + cur);
    }
    if (i < p.size()) cur.push_back(p[i]);
  }
  return RW_OK;
}

int write_all(int fd, const void* p, uint64_t n, const std::string& what) {
  const auto* b = static_cast<const uint8_t*>(p);
  while (n) {
    ssize_t w = ::write(fd, b, n > (1ull << 30) ? (1ull << 30) : n);
    if (w < 0) {
      if (errno == EINTR) continue;
      return cfail(RW_STORAGE_ERROR, "StorageError: short write on " + what);
    }
    b += w;
    n -= static_cast<uint64_t>(w);
  }
  return RW_OK;
}

int read_all(int fd, void* p, uint64_t n, uint64_t off, const std::string& what) {
  auto* b = static_cast<uint8_t*>(p);
  while (n) {
    ssize_t r = ::pread(fd, b, n > (1ull << 30) ? (1ull << 30) : n, static_cast<off_t>(off));
    if (r < 0 && errno == EINTR) continue;
    if (r <= 0) return cfail(RW_STORAGE_ERROR, "StorageError: short read on " + what);
    b += r;
    n -= static_cast<uint64_t>(r);
    off += static_cast<uint64_t>(r);
  }
  return RW_OK;
}

void fsync_dir(const std::string& d) {
  int fd = ::open(d.c_str(), O_RDONLY | O_DIRECTORY);
  if (fd >= 0) {
    ::fsync(fd);
    ::close(fd);
  }
}

// write_text_atomic (wire.cpp:140-142) + fsync so the rename is the commit
int write_text_atomic(const std::string& path, const std::string& text) {
  const std::string tmp = path + ".tmp";
  int fd = ::open(tmp.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
  if (fd < 0) return cfail(RW_STORAGE_ERROR, "StorageError: cannot open " + tmp);
  int st = write_all(fd, text.data(), text.size(), tmp);
  if (!st && ::fsync(fd) != 0) st = cfail(RW_STORAGE_ERROR, "StorageError: fsync failed on " + tmp);
  ::close(fd);
  if (st) return st;
  if (std::rename(tmp.c_str(), path.c_str()) != 0) return cfail(RW_STORAGE_ERROR, "StorageError: rename " + tmp);
  const size_t slash = path.rfind('/');
  fsync_dir(slash == std::string::npos ? "." : path.substr(0, slash));
  return RW_OK;
}

bool read_text(const std::string& path, std::string* out) {
  FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) return false;
  out->clear();
  char b[4096];
  size_t n;
  while ((n = std::fread(b, 1, sizeof(b), f)) > 0) out->append(b, n);
  std::fclose(f);
  return true;
}

struct BlobEntry {
  uint64_t bytes = 0;
  uint32_t crc = 0;
  uint32_t parts = 0;  // 0: one file <name>.bin; else <name>.bin.<k>, k < parts
};

// worker manifest: "SWCK 1\niteration I\nworker W\nblob <name> <bytes> <crc hex>\n...end\n"
bool parse_worker_manifest(const std::string& text, uint64_t it, uint32_t w, std::map<std::string, BlobEntry>* out) {
  out->clear();
  size_t pos = 0;
  bool header = false, ended = false, saw_it = false, saw_w = false;
  while (pos < text.size()) {
    size_t nl = text.find('\n', pos);
    if (nl == std::string::npos) return false;  // every line is newline-terminated
    const std::string line = text.substr(pos, nl - pos);
    pos = nl + 1;
    char name[256];
    unsigned long long a = 0, b = 0;
    unsigned crc = 0;
    if (!header) {
      if (line != "SWCK 1") return false;
      header = true;
    } else if (std::sscanf(line.c_str(), "iteration %llu", &a) == 1 && line.rfind("iteration ", 0) == 0) {
      if (a != it) return false;
      saw_it = true;
    } else if (std::sscanf(line.c_str(), "worker %llu", &b) == 1 && line.rfind("worker ", 0) == 0) {
      if (b != w) return false;
      saw_w = true;
    } else if (std::sscanf(line.c_str(), "blob %255s %llu %x", name, &a, &crc) == 3) {
      unsigned parts = 0;
      char n2[256];
      unsigned long long a2 = 0;
      unsigned c2 = 0;
      if (std::sscanf(line.c_str(), "blob %255s %llu %x %u", n2, &a2, &c2, &parts) != 4) parts = 0;
      (*out)[name] = BlobEntry{a, crc, parts};
    } else if (line == "end") {
      ended = true;
      break;
    } else {
      return false;
    }
  }
  return header && ended && saw_it && saw_w;
}

bool parse_global_manifest(const std::string& text, uint64_t it, uint32_t* workers) {
  unsigned long long a = 0, w = 0;
  if (std::sscanf(text.c_str(), "SWCK-MANIFEST 1\niteration %llu\nworkers %llu\n", &a, &w) != 2) return false;
  if (a != it || text.size() < 4 || text.compare(text.size() - 4, 4, "end\n") != 0) return false;
  if (workers) *workers = static_cast<uint32_t>(w);
  return true;
}

int first_device_blob(const rw_blob* blobs, uint32_t n) {
  for (uint32_t i = 0; blobs && i < n; ++i)
    if (!blobs[i].on_host && blobs[i].bytes) return rwb::DeviceScope::device_of(blobs[i].data);
  return -1;
}

}  // namespace

extern "C" {

int rw_ckpt_write(const char* dir, uint64_t iteration, uint32_t worker, const rw_blob* blobs, uint32_t n,
                  uint32_t crash_after_blobs, void* stream) {
  rwb::DeviceScope dev_scope(first_device_blob(blobs, n));
  if (!dir || (n && !blobs)) return cfail(RW_INVALID_ARGUMENT, "null argument");
  for (uint32_t i = 0; i < n; ++i) {
    if (!valid_name(blobs[i].name)) return cfail(RW_INVALID_ARGUMENT, "blob names are [A-Za-z0-9._-]+");
    if (blobs[i].bytes && !blobs[i].data) return cfail(RW_INVALID_ARGUMENT, "null blob data");
    for (uint32_t j = 0; j < i; ++j)
      if (std::strcmp(blobs[i].name, blobs[j].name) == 0) return cfail(RW_INVALID_ARGUMENT, "duplicate blob name");
  }
  const std::string wdir = worker_dir(dir, iteration, worker);
  int st = mkdirs(wdir);
  if (st) return st;
  bool any_dev = false;
  for (uint32_t i = 0; i < n; ++i) any_dev |= !blobs[i].on_host && blobs[i].bytes > 0;
  std::unique_lock<std::mutex> lk(g_ring.mu);
  if (any_dev) {
    st = ring_ready(g_ring);
    if (st) return st;
  }
  auto cs = static_cast<cudaStream_t>(stream);
  std::string wm = "SWCK 1\n";
  wm += "iteration " + std::to_string(iteration) + "\nworker " + std::to_string(worker) + "\n";
  for (uint32_t i = 0; i < n; ++i) {
    if (i == crash_after_blobs)  // test hook: simulated crash mid-write (no manifest)
      return cfail(RW_STORAGE_ERROR, "StorageError: injected crash during checkpoint write");
    const rw_blob& b = blobs[i];
    const std::string path = wdir + "/" + b.name + ".bin";
    uint32_t crc = 0, nparts = 0;
    if (b.on_host || b.bytes == 0) {
      int fd = ::open(path.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
      if (fd < 0) return cfail(RW_STORAGE_ERROR, "StorageError: cannot open " + path);
      crc = crc32_host(b.data, b.bytes);
      st = write_all(fd, b.data, b.bytes, path);
      if (!st && ::fsync(fd) != 0) st = cfail(RW_STORAGE_ERROR, "StorageError: fsync failed on " + path);
      ::close(fd);
    } else {
      nparts = parts_for(b.bytes);
      std::vector<int> fds;
      for (uint32_t w = 0; w < nparts && !st; ++w) {
        const int fd = ::open(part_path(path, w).c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
        if (fd < 0) st = cfail(RW_STORAGE_ERROR, "StorageError: cannot open " + part_path(path, w));
        else fds.push_back(fd);
      }
      if (!st) st = device_crc(g_ring, b.data, b.bytes, cs, &crc);
      if (!st) st = staged_io(g_ring, true, fds, b.data, b.bytes, cs, path);
      for (int fd : fds) ::close(fd);
    }
    if (st) return st;
    char line[320];
    std::snprintf(line, sizeof(line), "blob %s %llu %08x %u\n", b.name, static_cast<unsigned long long>(b.bytes),
                  crc, nparts);
    wm += line;
  }
  wm += "end\n";
  fsync_dir(wdir);
  char wb[32];
  std::snprintf(wb, sizeof(wb), "/w%05u.wm", worker);
  return write_text_atomic(iter_dir(dir, iteration) + wb, wm);
}

int rw_ckpt_commit(const char* dir, uint64_t iteration, uint32_t n_workers) {
  if (!dir || n_workers == 0) return cfail(RW_INVALID_ARGUMENT, "bad argument");
  for (uint32_t w = 0; w < n_workers; ++w) {
    char wb[32];
    std::snprintf(wb, sizeof(wb), "/w%05u.wm", w);
    std::string text;
    std::map<std::string, BlobEntry> m;
    if (!read_text(iter_dir(dir, iteration) + wb, &text) || !parse_worker_manifest(text, iteration, w, &m))
      return cfail(RW_STORAGE_ERROR, "StorageError: worker " + std::to_string(w) + " has not committed iteration " +
                                         std::to_string(iteration));
  }
  std::string g = "SWCK-MANIFEST 1\niteration " + std::to_string(iteration) + "\nworkers " +
                  std::to_string(n_workers) + "\nend\n";
  return write_text_atomic(manifest_path(dir, iteration), g);
}

int rw_ckpt_latest(const char* dir, uint64_t* iteration) {
  if (!dir || !iteration) return cfail(RW_INVALID_ARGUMENT, "null argument");
  DIR* d = ::opendir(dir);
  if (!d) return cfail(RW_NO_CHECKPOINT, std::string("NoCheckpoint: no checkpoint directory ") + dir);
  bool found = false;
  uint64_t best = 0;
  while (dirent* e = ::readdir(d)) {
    unsigned long long it = 0;
    char tail = 0;
    if (std::sscanf(e->d_name, "MANIFEST_%16llu%c", &it, &tail) != 1) continue;  // skips *.tmp
    if (std::strlen(e->d_name) != 9 + 16) continue;
    std::string text;
    if (!read_text(std::string(dir) + "/" + e->d_name, &text) || !parse_global_manifest(text, it, nullptr)) continue;
    if (!found || it > best) best = it;
    found = true;
  }
  ::closedir(d);
  if (!found) return cfail(RW_NO_CHECKPOINT, std::string("NoCheckpoint: no committed manifest in ") + dir);
  *iteration = best;
  return RW_OK;
}

int rw_ckpt_blob_bytes(const char* dir, uint64_t iteration, uint32_t worker, const char* name, uint64_t* bytes) {
  if (!dir || !name || !bytes) return cfail(RW_INVALID_ARGUMENT, "null argument");
  std::string text;
  if (!read_text(manifest_path(dir, iteration), &text) || !parse_global_manifest(text, iteration, nullptr))
    return cfail(RW_NO_CHECKPOINT, "NoCheckpoint: iteration " + std::to_string(iteration) + " not committed");
  char wb[32];
  std::snprintf(wb, sizeof(wb), "/w%05u.wm", worker);
  std::map<std::string, BlobEntry> m;
  if (!read_text(iter_dir(dir, iteration) + wb, &text) || !parse_worker_manifest(text, iteration, worker, &m))
    return cfail(RW_STORAGE_ERROR, "StorageError: bad worker manifest");
  auto it = m.find(name);
  if (it == m.end()) return cfail(RW_STORAGE_ERROR, std::string("StorageError: no blob ") + name);
  *bytes = it->second.bytes;
  return RW_OK;
}

int rw_ckpt_load(const char* dir, uint64_t iteration, uint32_t worker, const rw_blob* blobs, uint32_t n,
                 void* stream) {
  rwb::DeviceScope dev_scope(first_device_blob(blobs, n));
  if (!dir || (n && !blobs)) return cfail(RW_INVALID_ARGUMENT, "null argument");
  std::string text;
  uint32_t workers = 0;
  if (!read_text(manifest_path(dir, iteration), &text) || !parse_global_manifest(text, iteration, &workers))
    return cfail(RW_NO_CHECKPOINT, "NoCheckpoint: iteration " + std::to_string(iteration) + " not committed");
  if (worker >= workers) return cfail(RW_NO_CHECKPOINT, "NoCheckpoint: no such worker in the manifest");
  char wb[32];
  std::snprintf(wb, sizeof(wb), "/w%05u.wm", worker);
  std::map<std::string, BlobEntry> m;
  if (!read_text(iter_dir(dir, iteration) + wb, &text) || !parse_worker_manifest(text, iteration, worker, &m))
    return cfail(RW_STORAGE_ERROR, "StorageError: bad worker manifest");
  for (uint32_t i = 0; i < n; ++i) {  // every check before any byte moves
    if (!valid_name(blobs[i].name)) return cfail(RW_INVALID_ARGUMENT, "bad blob name");
    auto it = m.find(blobs[i].name);
    if (it == m.end()) return cfail(RW_STORAGE_ERROR, std::string("StorageError: no blob ") + blobs[i].name);
    if (it->second.bytes != blobs[i].bytes)
      return cfail(RW_SHAPE_MISMATCH, std::string("ShapeMismatch: blob ") + blobs[i].name + " size differs");
    if (blobs[i].bytes && !blobs[i].data) return cfail(RW_INVALID_ARGUMENT, "null blob data");
  }
  bool any_dev = false;
  for (uint32_t i = 0; i < n; ++i) any_dev |= !blobs[i].on_host && blobs[i].bytes > 0;
  std::unique_lock<std::mutex> lk(g_ring.mu);
  int st = RW_OK;
  if (any_dev) {
    st = ring_ready(g_ring);
    if (st) return st;
  }
  auto cs = static_cast<cudaStream_t>(stream);
  const std::string wdir = worker_dir(dir, iteration, worker);
  for (uint32_t i = 0; i < n; ++i) {
    const rw_blob& b = blobs[i];
    const BlobEntry& ent = m[b.name];
    const std::string path = wdir + "/" + b.name + ".bin";
    const uint32_t nfiles = ent.parts ? ent.parts : 1;
    std::vector<int> fds;
    for (uint32_t w = 0; w < nfiles && !st; ++w) {
      const std::string fp = ent.parts ? part_path(path, w) : path;
      const uint64_t want = ent.parts ? part_bytes(ent.bytes, ent.parts, w) : ent.bytes;
      const int fd = ::open(fp.c_str(), O_RDONLY);
      struct stat sb;
      if (fd < 0) {
        st = cfail(RW_STORAGE_ERROR, "StorageError: cannot open " + fp);
      } else {
        fds.push_back(fd);
        if (::fstat(fd, &sb) != 0 || static_cast<uint64_t>(sb.st_size) != want)
          st = cfail(RW_STORAGE_ERROR, "StorageError: truncated blob " + fp);
      }
    }
    uint32_t crc = 0;
    if (st) {
    } else if (!ent.parts) {  // single file: host blob or a device blob written as one
      if (b.on_host) {
        st = read_all(fds[0], b.data, b.bytes, 0, path);
        if (!st) crc = crc32_host(b.data, b.bytes);
      } else if (b.bytes) {
        st = staged_io(g_ring, false, fds, b.data, b.bytes, cs, path);
        if (!st) st = device_crc(g_ring, b.data, b.bytes, cs, &crc);
      }
    } else if (b.on_host) {  // device-written parts into a host buffer
      uint64_t off = 0;
      for (uint32_t w = 0; w < ent.parts && !st; ++w) {
        const uint64_t pb = part_bytes(ent.bytes, ent.parts, w);
        st = read_all(fds[w], static_cast<char*>(b.data) + off, pb, 0, part_path(path, w));
        off += pb;
      }
      if (!st) crc = crc32_host(b.data, b.bytes);
    } else {
      st = staged_io(g_ring, false, fds, b.data, b.bytes, cs, path);
      if (!st) st = device_crc(g_ring, b.data, b.bytes, cs, &crc);
    }
    for (int fd : fds) ::close(fd);
    if (st) return st;
    if (crc != ent.crc) return cfail(RW_STORAGE_ERROR, "StorageError: checksum mismatch in " + path);
  }
  return RW_OK;
}

// gc_logs: remove every committed log chunk whose records all
// belong to iterations < ckpt_iteration; requires that checkpoint committed.
int rw_log_gc(const char* log_dir, const char* ckpt_dir, uint64_t ckpt_iteration, uint32_t* deleted) {
  if (!log_dir || !ckpt_dir || !deleted) return cfail(RW_INVALID_ARGUMENT, "null argument");
  *deleted = 0;
  std::string text;
  if (!read_text(manifest_path(ckpt_dir, ckpt_iteration), &text) ||
      !parse_global_manifest(text, ckpt_iteration, nullptr))
    return cfail(RW_NO_CHECKPOINT, "NoCheckpoint: gc needs a committed checkpoint at iteration " +
                                       std::to_string(ckpt_iteration));
  DIR* d = ::opendir(log_dir);
  if (!d) return RW_OK;  // nothing logged yet
  std::vector<std::string> names;
  while (dirent* e = ::readdir(d)) {
    const std::string nm = e->d_name;
    if (nm.size() > 5 && nm.compare(nm.size() - 5, 5, ".swft") == 0) names.push_back(nm);
  }
  ::closedir(d);
  std::sort(names.begin(), names.end());
  for (const std::string& nm : names) {
    const std::string path = std::string(log_dir) + "/" + nm;
    rw_log_reader* r = nullptr;
    if (rw_log_open(&r, path.c_str(), nullptr) != RW_OK) continue;  // not ours / corrupt: keep
    bool keep = false, bad = false;
    for (;;) {
      rw_log_record rec;
      int32_t eof = 0;
      if (rw_log_skip(r, &rec, &eof) != RW_OK) {
        bad = true;
        break;
      }
      if (eof) break;
      if (rec.iteration >= ckpt_iteration) {
        keep = true;
        break;
      }
    }
    rw_log_close(r);
    if (keep || bad) continue;
    if (std::remove(path.c_str()) == 0) ++*deleted;
  }
  return RW_OK;
}

}  // extern "C"

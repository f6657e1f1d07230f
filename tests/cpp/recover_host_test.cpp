// Multi-process C++ host of the whole Swift recovery path, through the C ABI
// only (no Python, no torch): one process per GPU, NCCL communicators from a
// ncclUniqueId the launcher shares before fork (the "file bootstrap").
//
//   recover_host_test replication <nranks> [gpt2xl]
//       rank 0 crashed mid-update (MidUpdate(G/2)), ranks 1.. are
//       replacements: rw_resolve (replacements join with no state) ->
//       rw_recover_replication (pipelined undo + NCCL broadcast).  Every rank's
//       x, m, v, markers must equal a local single-GPU rw_apply_resolution of
//       the same crash bit for bit (CRC32 compared across ranks).
//   recover_host_test replay <nranks>
//       rw_recover_parallel of a 2-stage group over the ranks vs
//       rw_replay_group on one GPU: bit-identical x, m, v.
//   recover_host_test failure <nranks>
//       the last rank dies (fail-stop) before a collective; survivors detect it
//       (rw_comm_watch timeout + heartbeat membership), shrink the communicator
//       (ncclCommShrink with NCCL_SHRINK_ABORT), resolve among themselves; a
//       replacement process then joins a fresh communicator and receives the
//       resolved state (rw_recover_replication).  Prints detect / shrink /
//       join / recovery times.
//
// Prints "PASS <scenario> ..." lines and exits 0 iff every check held.
#include <cuda_runtime.h>
#include <signal.h>
#include <sys/stat.h>
#include <sys/wait.h>
#include <unistd.h>

#include <array>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "rewind_b200.h"

using Clock = std::chrono::steady_clock;
static double ms_since(Clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

static int g_fail = 0;
#define EXPECT(cond, ...)                     \
  do {                                        \
    if (!(cond)) {                            \
      std::printf("FAIL rank %d: ", g_rank);  \
      std::printf(__VA_ARGS__);               \
      std::printf("\n");                      \
      ++g_fail;                               \
    }                                         \
  } while (0)
#define CK(call)                                                                               \
  do {                                                                                         \
    int st_ = (call);                                                                          \
    if (st_) {                                                                                 \
      std::printf("FAIL rank %d: %s -> %d (%s)\n", g_rank, #call, st_, rw_last_error_message()); \
      std::fflush(stdout);                                                                     \
      _exit(3);                                                                                \
    }                                                                                          \
  } while (0)
#define CU(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) {                                                              \
      std::printf("FAIL rank %d: %s -> %s\n", g_rank, #call, cudaGetErrorString(e_));     \
      _exit(3);                                                                           \
    }                                                                                     \
  } while (0)

static int g_rank = -1;
static const Clock::time_point g_t0 = Clock::now();
// progress trace (stderr, timestamped): where a multi-process scenario is
#define TRACE(...)                                                              \
  do {                                                                          \
    std::fprintf(stderr, "[%8.1f ms] rank %d: ", ms_since(g_t0), g_rank);       \
    std::fprintf(stderr, __VA_ARGS__);                                          \
    std::fprintf(stderr, "\n");                                                \
  } while (0)

// ---------------------------------------------------------------- layouts
static std::vector<uint64_t> gpt2_xl_sizes() {  // 1,557,611,200 params, 580 groups (workloads.py)
  const uint64_t D = 1600, L = 48, V = 50257, P = 1024;
  std::vector<uint64_t> s = {V * D, P * D};
  for (uint64_t l = 0; l < L; ++l)
    for (uint64_t v : {D, D, D * 3 * D, 3 * D, D * D, D, D, D, D * 4 * D, 4 * D, 4 * D * D, D}) s.push_back(v);
  s.push_back(D);
  s.push_back(D);
  return s;
}
static std::vector<uint64_t> small_sizes() {
  std::vector<uint64_t> s;
  for (int i = 0; i < 40; ++i) s.push_back(1000 + 977 * uint64_t(i % 7) + (i % 3 ? 3 : 4096));
  return s;
}

struct Flat {
  std::vector<rw_group> groups;
  uint64_t total = 0;
  float *x = nullptr, *g = nullptr, *m = nullptr, *v = nullptr;
  rw_state* st = nullptr;
};
static Flat make_flat(const std::vector<uint64_t>& sizes, int device) {
  Flat f;
  for (uint64_t n : sizes) {
    rw_group g{};
    g.offset = f.total;
    g.len = n;
    f.groups.push_back(g);
    f.total += (n + 63) / 64 * 64;
  }
  CU(cudaMalloc(&f.x, f.total * 4));
  CU(cudaMalloc(&f.g, f.total * 4));
  CU(cudaMalloc(&f.m, f.total * 4));
  CU(cudaMalloc(&f.v, f.total * 4));
  CU(cudaMemset(f.x, 0, f.total * 4));
  CU(cudaMemset(f.g, 0, f.total * 4));
  CU(cudaMemset(f.m, 0, f.total * 4));
  CU(cudaMemset(f.v, 0, f.total * 4));
  CK(rw_state_create(&f.st, RW_F32, f.x, f.g, f.m, f.v, nullptr, f.total, f.groups.data(),
                     uint32_t(f.groups.size()), device));
  return f;
}
static void free_flat(Flat& f) {
  rw_state_destroy(f.st);
  cudaFree(f.x), cudaFree(f.g), cudaFree(f.m), cudaFree(f.v);
}
static rw_hyper adam() {
  rw_hyper h{};
  h.kind = RW_ADAM;
  h.lr = 1e-4;
  h.weight_decay = 0.01;
  h.beta1 = 0.9;
  h.beta2 = 0.999;
  h.eps = 1e-8;
  h.momentum = 0.9;
  return h;
}
// seeded Adam state at t = 10 (x, g, m, v from rw_seeded_fill), as bench.py's _fill_adam_state
static void fill_state(Flat& f) {
  CK(rw_seeded_fill(RW_F32, f.x, f.total, 2302, 0, nullptr));
  CK(rw_seeded_fill(RW_F32, f.g, f.total, 2303, 0, nullptr));
  CK(rw_seeded_fill(RW_F32, f.m, f.total, 2304, 0, nullptr));
  CK(rw_seeded_fill(RW_F32, f.v, f.total, 2305, 0, nullptr));
  // m *= 0.01; v = |v| * 1e-4 : host round trip keeps this file kernel-free
  std::vector<float> h(f.total);
  CU(cudaMemcpy(h.data(), f.m, f.total * 4, cudaMemcpyDeviceToHost));
  for (float& z : h) z *= 0.01f;
  CU(cudaMemcpy(f.m, h.data(), f.total * 4, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(h.data(), f.v, f.total * 4, cudaMemcpyDeviceToHost));
  for (float& z : h) z = std::fabs(z) * 1e-4f;
  CU(cudaMemcpy(f.v, h.data(), f.total * 4, cudaMemcpyHostToDevice));
  std::vector<rw_group> mk = f.groups;
  for (auto& g : mk) g.t = 10, g.updated = 0;
  CK(rw_state_write_groups(f.st, mk.data(), nullptr));
}
static void crash(Flat& f, const rw_hyper& h, uint32_t k) {  // MidUpdate(k), update order = reverse layer order
  const uint32_t G = uint32_t(f.groups.size());
  std::vector<uint32_t> ids(G);
  for (uint32_t i = 0; i < G; ++i) ids[i] = G - 1 - i;
  CK(rw_optimizer_step(f.st, &h, ids.data(), G, nullptr, k, nullptr));
  CU(cudaDeviceSynchronize());
}
static uint32_t crc_of(const void* p, uint64_t bytes) {
  uint32_t* d = nullptr;
  CU(cudaMalloc(&d, 4));
  CK(rw_crc32_device(p, bytes, d, nullptr));
  uint32_t h = 0;
  CU(cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost));
  cudaFree(d);
  return h;
}
static bool same_device(const void* a, const void* b, uint64_t bytes) {
  std::vector<char> ha(bytes), hb(bytes);
  CU(cudaMemcpy(ha.data(), a, bytes, cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(hb.data(), b, bytes, cudaMemcpyDeviceToHost));
  return std::memcmp(ha.data(), hb.data(), bytes) == 0;
}
static std::vector<rw_group> markers(Flat& f) {
  std::vector<rw_group> mk(f.groups.size());
  CK(rw_state_read_groups(f.st, mk.data(), nullptr));
  return mk;
}

// all ranks' CRCs through the communicator itself: an all-gather built from
// the ordered reduce (rank r contributes "micro-batch" r holding its CRC as
// two exact 16-bit halves; every other slot is zero, so the sums are exact)
static std::vector<uint32_t> gather_u32(rw_comm* c, uint32_t mine) {
  const int n = rw_comm_size(c), r = rw_comm_rank(c);
  const uint64_t len = 2 * uint64_t(n);
  const uint64_t out_elems = rw_ordered_reduce_out_elems(len, n);
  float *part = nullptr, *out = nullptr, *scr = nullptr;
  CU(cudaMalloc(&part, len * 4));
  CU(cudaMalloc(&out, out_elems * 4));
  const uint64_t se = rw_ordered_reduce_scratch_elems(len, uint32_t(n), n, r);
  CU(cudaMalloc(&scr, (se ? se : 1) * 4));
  std::vector<float> h(len, 0.f);
  h[2 * uint64_t(r)] = float(mine & 0xFFFFu);
  h[2 * uint64_t(r) + 1] = float(mine >> 16);
  CU(cudaMemcpy(part, h.data(), len * 4, cudaMemcpyHostToDevice));
  std::vector<const float*> parts(uint64_t(n), nullptr);
  parts[uint64_t(r)] = part;  // micro-batch r belongs to rank r (r mod n == r)
  CK(rw_ordered_reduce(c, parts.data(), uint32_t(n), len, out, scr, se, nullptr));
  CU(cudaDeviceSynchronize());
  CU(cudaMemcpy(h.data(), out, len * 4, cudaMemcpyDeviceToHost));
  cudaFree(part), cudaFree(out), cudaFree(scr);
  std::vector<uint32_t> all(static_cast<size_t>(n), 0u);
  for (int q = 0; q < n; ++q) all[size_t(q)] = uint32_t(h[2 * q]) | (uint32_t(h[2 * q + 1]) << 16);
  return all;
}

// ------------------------------------------------------------- replication
static int run_replication(int rank, int n, const void* id, bool big, uint32_t flags) {
  CU(cudaSetDevice(rank));
  rw_comm* c = nullptr;
  CK(rw_comm_init(&c, id, n, rank, rank));
  const auto sizes = big ? gpt2_xl_sizes() : small_sizes();
  const uint32_t G = uint32_t(sizes.size());
  rw_hyper h = adam();
  Flat f = make_flat(sizes, rank);
  Flat expect{};
  std::array<uint32_t, 3> exp_crc{};
  if (rank == 0) {
    fill_state(f);
    crash(f, h, G / 2);
    // the same crash repaired locally on one GPU: the expected result
    expect = make_flat(sizes, rank);
    fill_state(expect);
    crash(expect, h, G / 2);
    std::vector<uint8_t> acts(G);
    rw_resolution rs{};
    // a 1-rank resolve equals the local plan: use the summary functions directly
    std::vector<rw_group> mk = markers(expect);
    rw_resolve_summary loc{}, glob{};
    CK(rw_resolve_summarize(mk.data(), G, nullptr, &h, UINT64_MAX, &loc));
    CK(rw_resolve_summarize(mk.data(), G, nullptr, &h, loc.t_min, &glob));
    uint64_t tgt = 0;
    int32_t strat = 0;
    CK(rw_resolve_plan(&glob, RW_POLICY_UNDO, mk.data(), G, acts.data(), &tgt, &strat));
    CK(rw_apply_resolution(expect.st, &h, acts.data(), strat, nullptr, nullptr));
    CU(cudaDeviceSynchronize());
    (void)rs;
    // keep only its CRCs: a second resident copy of the state would also crowd
    // the survivor's address translation during the timed transfer
    const uint64_t nbe = expect.total * 4;
    exp_crc = {crc_of(expect.x, nbe), crc_of(expect.m, nbe), crc_of(expect.v, nbe)};
    free_flat(expect);
  }
  CU(cudaDeviceSynchronize());
  cudaStream_t s;
  CU(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  // warm-up exchange (connections, and for the chain the IPC mappings, which a
  // communicator keeps), then the timed recovery
  {
    rw_resolution w{};
    std::vector<uint8_t> a(G);
    CK(rw_resolve(rank == 0 ? f.st : nullptr, &h, c, RW_POLICY_UNDO, nullptr, rank == 0 ? a.data() : nullptr, &w, s));
    std::vector<uint8_t> none(G, 0);  // transfers without undo: the survivor's state is left as it is
    uint64_t wb = 0;
    for (int w = 0; w < 3; ++w) {
      CK(rw_recover_replication(f.st, &h, c, 0, rank == 0 ? none.data() : nullptr, RW_STRATEGY_NONE, flags, 16, s,
                                &wb));
      CU(cudaStreamSynchronize(s));
    }
  }
  const auto t0 = Clock::now();
  std::vector<uint8_t> acts(G, 0);
  rw_resolution res{};
  CK(rw_resolve(rank == 0 ? f.st : nullptr, &h, c, RW_POLICY_UNDO, nullptr, rank == 0 ? acts.data() : nullptr, &res,
                s));
  const double t_resolve = ms_since(t0);
  uint64_t bytes = 0;
  CK(rw_recover_replication(f.st, &h, c, 0, rank == 0 ? acts.data() : nullptr, res.strategy, flags, 16, s, &bytes));
  CU(cudaStreamSynchronize(s));
  const double t_total = ms_since(t0);
  EXPECT(res.strategy == RW_STRATEGY_UNDO && res.target == 10, "plan %d target %llu", res.strategy,
         (unsigned long long)res.target);
  const uint64_t nb = f.total * 4;
  const uint32_t cx = crc_of(f.x, nb), cm = crc_of(f.m, nb), cv = crc_of(f.v, nb);
  if (rank == 0) {
    EXPECT(cx == exp_crc[0] && cm == exp_crc[1] && cv == exp_crc[2], "survivor state != local rw_apply_resolution");
  }
  for (auto& g : markers(f)) EXPECT(g.t == 10 && g.updated == 0, "marker (%llu, %u)", (unsigned long long)g.t, g.updated);
  const auto all_x = gather_u32(c, cx), all_m = gather_u32(c, cm), all_v = gather_u32(c, cv);
  for (int r = 1; r < n; ++r)
    EXPECT(all_x[r] == all_x[0] && all_m[r] == all_m[0] && all_v[r] == all_v[0], "rank %d CRC differs", r);
  if (rank == 0)
    std::printf("PASS replication%s n=%d groups=%u bytes_per_replacement=%llu resolve_ms=%.3f recovery_ms=%.3f "
                "(%.1f GB/s per replacement)\n",
                (flags & RW_RECOVER_CHAIN) ? " (copy-engine chain)" : "", n, G, (unsigned long long)bytes,
                t_resolve, t_total, bytes / (t_total * 1e-3) / 1e9);
  free_flat(f);
  CK(rw_comm_destroy(c));
  return g_fail ? 1 : 0;
}

// ------------------------------------------------------------------ replay
struct StageBufs {
  std::vector<int64_t> dims;
  std::vector<rw_group> groups;
  uint64_t total = 0;
  float *x = nullptr, *g = nullptr, *m = nullptr, *v = nullptr, *grad = nullptr;
  rw_state* st = nullptr;
  std::vector<void*> w16;
  std::vector<const void*> wc;
  std::vector<const float*> b;
  rw_replay_stage rs{};
};
static void make_stage(StageBufs& S, int sid, std::vector<int64_t> dims, int device) {
  S.dims = dims;
  const int L = int(dims.size()) - 1;
  for (int l = 0; l < L; ++l)
    for (uint64_t n : {uint64_t(dims[l] * dims[l + 1]), uint64_t(dims[l + 1])}) {
      rw_group g{};
      g.offset = S.total;
      g.len = n;
      S.groups.push_back(g);
      S.total += (n + 63) / 64 * 64;
    }
  for (float** p : {&S.x, &S.g, &S.m, &S.v, &S.grad}) {
    CU(cudaMalloc(p, S.total * 4));
    CU(cudaMemset(*p, 0, S.total * 4));
  }
  CK(rw_state_create(&S.st, RW_F32, S.x, S.g, S.m, S.v, nullptr, S.total, S.groups.data(),
                     uint32_t(S.groups.size()), device));
  for (int l = 0; l < L; ++l) {  // make_stage (model.cpp:45-50): W from {id, l, 0}, b from {id, l, 1}
    const uint64_t pw[3] = {uint64_t(sid), uint64_t(l), 0}, pb[3] = {uint64_t(sid), uint64_t(l), 1};
    CK(rw_seeded_fill(RW_F32, S.x + S.groups[2 * l].offset, S.groups[2 * l].len, rw_derive_seed(7, pw, 3), 0, nullptr));
    CK(rw_seeded_fill(RW_F32, S.x + S.groups[2 * l + 1].offset, S.groups[2 * l + 1].len, rw_derive_seed(7, pb, 3), 0,
                      nullptr));
    void* w = nullptr;
    CU(cudaMalloc(&w, S.groups[2 * l].len * 2));
    CK(rw_cast_f32_to_bf16(S.x + S.groups[2 * l].offset, w, S.groups[2 * l].len, nullptr));
    S.w16.push_back(w);
    S.wc.push_back(w);
    S.b.push_back(S.x + S.groups[2 * l + 1].offset);
  }
  S.rs.desc.num_layers = L;
  S.rs.desc.dims = S.dims.data();
  S.rs.desc.w = S.wc.data();
  S.rs.desc.b = S.b.data();
  S.rs.state = S.st;
  S.rs.grad = S.grad;
}
static void free_stage(StageBufs& S) {
  rw_state_destroy(S.st);
  for (float* p : {S.x, S.g, S.m, S.v, S.grad}) cudaFree(p);
  for (void* w : S.w16) cudaFree(w);
}

static int run_replay(int rank, int n, const void* id) {
  CU(cudaSetDevice(rank));
  rw_comm* c = nullptr;
  CK(rw_comm_init(&c, id, n, rank, rank));
  const std::vector<int64_t> dims = {256, 1024, 256};
  const int64_t R = 384;
  const uint32_t m = 4, iters = 2;
  rw_hyper h = adam();
  h.lr = 1e-3;
  // the group's inbound log: activations into stage 0 and gradients into stage 1
  std::vector<void*> acts(iters * m), grads(iters * m);
  for (uint32_t i = 0; i < iters * m; ++i) {
    CU(cudaMalloc(&acts[i], R * dims[0] * 2));
    CU(cudaMalloc(&grads[i], R * dims[2] * 2));
    CK(rw_seeded_fill(RW_BF16, acts[i], R * dims[0], 1000 + i, 0, nullptr));
    CK(rw_seeded_fill(RW_BF16, grads[i], R * dims[2], 2000 + i, 0, nullptr));
  }
  rw_replay_log log{};
  log.acts = const_cast<const void* const*>(acts.data());
  log.grads = const_cast<const void* const*>(grads.data());
  log.seed = 7;
  StageBufs par[2], seq[2];
  for (int k = 0; k < 2; ++k) make_stage(par[k], 1 + k, dims, rank), make_stage(seq[k], 1 + k, dims, rank);
  rw_replay_stage ps[2] = {par[0].rs, par[1].rs}, ss[2] = {seq[0].rs, seq[1].rs};
  const uint64_t wpar = rw_replay_workspace_bytes(ps, 2, R, m, c), wseq = rw_replay_workspace_bytes(ss, 2, R, m, nullptr);
  EXPECT(wpar > 0 && wseq > 0, "workspace sizes");
  void *wp = nullptr, *wq = nullptr;
  CU(cudaMalloc(&wp, wpar));
  CU(cudaMalloc(&wq, wseq));
  CK(rw_recover_parallel(ps, 2, R, m, 5, 5 + iters, &h, &log, c, wp, wpar, nullptr));
  CK(rw_replay_group(ss, 2, R, m, 5, 5 + iters, &h, &log, wq, wseq, nullptr));
  CU(cudaDeviceSynchronize());
  for (int k = 0; k < 2; ++k) {
    const uint64_t nb = par[k].total * 4;
    EXPECT(same_device(par[k].x, seq[k].x, nb) && same_device(par[k].m, seq[k].m, nb) &&
               same_device(par[k].v, seq[k].v, nb),
           "stage %d: parallel != sequential", k);
    auto mk = std::vector<rw_group>(par[k].groups.size());
    CK(rw_state_read_groups(par[k].st, mk.data(), nullptr));
    for (auto& g : mk) EXPECT(g.t == iters && g.updated == 0, "stage %d marker", k);
    const auto all = gather_u32(c, crc_of(par[k].x, nb));
    for (int r = 1; r < n; ++r) EXPECT(all[r] == all[0], "stage %d: rank %d x differs", k, r);
  }
  if (rank == 0) std::printf("PASS replay n=%d m=%u iterations=%u parallel == sequential bit for bit\n", n, m, iters);
  for (int k = 0; k < 2; ++k) free_stage(par[k]), free_stage(seq[k]);
  for (auto p : acts) cudaFree(p);
  for (auto p : grads) cudaFree(p);
  cudaFree(wp), cudaFree(wq);
  CK(rw_comm_destroy(c));
  return g_fail ? 1 : 0;
}

// ----------------------------------------------------------------- failure
static void write_file(const std::string& p, const void* data, size_t n) {
  const std::string tmp = p + ".tmp";
  FILE* f = std::fopen(tmp.c_str(), "wb");
  std::fwrite(data, 1, n, f);
  std::fclose(f);
  std::rename(tmp.c_str(), p.c_str());
}
static bool read_file(const std::string& p, void* data, size_t n) {
  FILE* f = std::fopen(p.c_str(), "rb");
  if (!f) return false;
  const size_t got = std::fread(data, 1, n, f);
  std::fclose(f);
  return got == n;
}

// waits for a file another rank publishes; a rank that failed before
// publishing must not leave this one spinning forever
static bool wait_file(const std::string& p, void* data, size_t n, double limit_ms = 60000.0) {
  const auto t0 = Clock::now();
  while (!read_file(p, data, n)) {
    if (ms_since(t0) > limit_ms) {
      TRACE("gave up waiting for %s after %.0f ms", p.c_str(), limit_ms);
      return false;
    }
    std::this_thread::sleep_for(std::chrono::milliseconds(1));
  }
  return true;
}

static int run_failure(int rank, int n, const void* id, const std::string& dir, bool replacement) {
  // survivors: ranks 0..n-2; the dying rank n-1; the replacement takes rank n-1 of a new communicator
  const int dev = replacement ? n - 1 : rank;
  CU(cudaSetDevice(dev));
  const auto sizes = small_sizes();
  const uint32_t G = uint32_t(sizes.size());
  rw_hyper h = adam();
  rw_membership* mem = nullptr;
  if (replacement) {  // join: wait for the survivors' new unique id, then take over the dead slot
    unsigned char nid[128];
    if (!wait_file(dir + "/join.id", nid, sizeof(nid))) return 1;
    CK(rw_membership_open(&mem, (dir + "/heartbeats").c_str(), n - 1, n, 2000));
    const auto t0 = Clock::now();
    rw_comm* c = nullptr;
    CK(rw_comm_init(&c, nid, n, n - 1, dev));
    CK(rw_comm_watch(c, 200, 10000));
    const double join_ms = ms_since(t0);
    TRACE("replacement joined in %.1f ms", join_ms);
    Flat f = make_flat(sizes, dev);
    rw_resolution res{};
    CK(rw_resolve(nullptr, &h, c, RW_POLICY_UNDO, nullptr, nullptr, &res, nullptr));
    uint64_t bytes = 0;
    CK(rw_recover_replication(f.st, &h, c, 0, nullptr, res.strategy, 0, 8, nullptr, &bytes));
    CU(cudaDeviceSynchronize());
    const uint64_t nb = f.total * 4;
    const auto all = gather_u32(c, crc_of(f.x, nb));
    for (int r = 1; r < n; ++r) EXPECT(all[r] == all[0], "after join: rank %d x differs", r);
    for (auto& g : markers(f)) EXPECT(g.t == 10 && g.updated == 0, "replacement marker");
    std::printf("replacement: join_ms=%.1f received %llu bytes\n", join_ms, (unsigned long long)bytes);
    free_flat(f);
    CK(rw_comm_destroy(c));
    rw_membership_close(mem);
    return g_fail ? 1 : 0;
  }
  CK(rw_membership_open(&mem, (dir + "/heartbeats").c_str(), rank, n, 2000));
  rw_comm* c = nullptr;
  CK(rw_comm_init(&c, id, n, rank, dev));
  CK(rw_comm_watch(c, 200, 1500));
  TRACE("communicator up");  // poll 200 us, a collective stuck for 1.5 s = a dead peer
  Flat f = make_flat(sizes, dev);
  fill_state(f);
  // a healthy exchange first
  std::vector<uint8_t> acts(G);
  rw_resolution res{};
  CK(rw_resolve(f.st, &h, c, RW_POLICY_UNDO, nullptr, acts.data(), &res, nullptr));
  EXPECT(res.strategy == RW_STRATEGY_NONE, "healthy plan");
  TRACE("healthy exchange done");
  if (rank == n - 1) {  // fail-stop in the middle of the next iteration's update
    crash(f, h, G / 3);
    std::fflush(stdout);
    _exit(0);
  }
  crash(f, h, G / 2);  // survivors torn at a different point
  const auto t_fail = Clock::now();
  int st = rw_resolve(f.st, &h, c, RW_POLICY_UNDO, nullptr, acts.data(), &res, nullptr);
  const double t_detect_wall = ms_since(t_fail);
  EXPECT(st == RW_CHANNEL_BROKEN, "resolve with a dead peer returned %d", st);
  TRACE("resolve failed as expected after %.1f ms: %s", t_detect_wall, rw_last_error_message());
  int32_t reason = 0;
  double detect_ms = 0;
  CK(rw_comm_failed(c, &reason, &detect_ms));
  EXPECT(reason == RW_COMM_FAILED_TIMEOUT || reason == RW_COMM_FAILED_NCCL_ERROR, "failure reason %d", reason);
  // who is gone: the heartbeat membership
  int32_t dead[8], nd = 0;
  const auto t_m = Clock::now();
  do {
    CK(rw_membership_dead(mem, 500, dead, 8, &nd));
    if (!nd) std::this_thread::sleep_for(std::chrono::milliseconds(5));
  } while (!nd && ms_since(t_m) < 5000);
  EXPECT(nd == 1 && dead[0] == n - 1, "membership saw %d dead", nd);
  TRACE("membership: %d dead", nd);
  // repair among the survivors: shrink, then the consensus over them
  const auto t_s = Clock::now();
  rw_comm* sc = nullptr;
  const char* repair = "ncclCommShrink";
  if (rw_comm_shrink(c, dead, nd, &sc) != RW_OK) {
    // fallback: a fresh communicator over the survivors (id from the lowest survivor)
    TRACE("shrink failed (%s); re-forming the survivors' communicator", rw_last_error_message());
    repair = "re-init";
    unsigned char sid[128];
    if (rank == 0) {
      CK(rw_nccl_unique_id(sid));
      write_file(dir + "/survivors.id", sid, sizeof(sid));
    } else {
      if (!wait_file(dir + "/survivors.id", sid, sizeof(sid))) return 1;
    }
    CK(rw_comm_init(&sc, sid, n - 1, rank, dev));
  }
  const double shrink_ms = ms_since(t_s);
  CK(rw_comm_watch(sc, 200, 10000));
  TRACE("survivor communicator (%s) in %.1f ms", repair, shrink_ms);
  CK(rw_comm_abort(c));
  EXPECT(rw_comm_size(sc) == n - 1, "shrunk size %d", rw_comm_size(sc));
  CK(rw_resolve(f.st, &h, sc, RW_POLICY_UNDO, nullptr, acts.data(), &res, nullptr));
  EXPECT(res.strategy == RW_STRATEGY_UNDO && res.target == 10, "survivor plan %d", res.strategy);
  CK(rw_apply_resolution(f.st, &h, acts.data(), res.strategy, nullptr, nullptr));
  CU(cudaDeviceSynchronize());
  TRACE("survivors resolved + undone");
  // the replacement joins a fresh communicator (survivors + replacement)
  unsigned char nid[128];
  if (rank == 0) {
    CK(rw_nccl_unique_id(nid));
    write_file(dir + "/join.id", nid, sizeof(nid));
  } else if (!wait_file(dir + "/join.id", nid, sizeof(nid))) {
    return 1;
  }
  const auto t_j = Clock::now();
  rw_comm* jc = nullptr;
  CK(rw_comm_init(&jc, nid, n, rank, dev));
  CK(rw_comm_watch(jc, 200, 10000));
  const double join_ms = ms_since(t_j);
  TRACE("joined in %.1f ms", join_ms);
  rw_resolution r2{};
  const auto t_r = Clock::now();
  CK(rw_resolve(f.st, &h, jc, RW_POLICY_UNDO, nullptr, acts.data(), &r2, nullptr));
  uint64_t bytes = 0;
  CK(rw_recover_replication(f.st, &h, jc, 0, rank == 0 ? acts.data() : nullptr, r2.strategy, 0, 8, nullptr, &bytes));
  CU(cudaDeviceSynchronize());
  const double rec_ms = ms_since(t_r);
  const uint64_t nb = f.total * 4;
  const auto all = gather_u32(jc, crc_of(f.x, nb));
  for (int r = 1; r < n; ++r) EXPECT(all[r] == all[0], "after join: rank %d x differs", r);
  if (rank == 0)
    std::printf("PASS failure n=%d detect_ms=%.1f (watchdog age %.1f, reason %d) survivors_comm=%s %.1f ms "
                "join_ms=%.1f resolve+recover_ms=%.2f\n",
                n, t_detect_wall, detect_ms, reason, repair, shrink_ms, join_ms, rec_ms);
  free_flat(f);
  CK(rw_comm_abort(sc));
  CK(rw_comm_destroy(jc));
  rw_membership_close(mem);
  return g_fail ? 1 : 0;
}

int main(int argc, char** argv) {
  if (argc < 3) {
    std::printf("usage: %s replication|replay|failure <nranks> [gpt2xl] [chain]\n", argv[0]);
    return 2;
  }
  const std::string what = argv[1];
  const int n = std::atoi(argv[2]);
  bool big = false;
  uint32_t rflags = 0;
  for (int a = 3; a < argc; ++a) {
    if (std::string(argv[a]) == "gpt2xl") big = true;
    if (std::string(argv[a]) == "chain") rflags |= RW_RECOVER_CHAIN;
  }
  unsigned char id[128];
  if (rw_nccl_unique_id(id)) {  // no CUDA context is created before fork
    std::printf("FAIL ncclGetUniqueId: %s\n", rw_last_error_message());
    return 1;
  }
  char tmpl[] = "/tmp/rw_host_XXXXXX";
  const std::string dir = mkdtemp(tmpl);
  std::vector<pid_t> kids;
  for (int r = 0; r < n; ++r) {
    const pid_t p = fork();
    if (p == 0) {
      g_rank = r;
      int rc = 0;
      if (what == "replication") rc = run_replication(r, n, id, big, rflags);
      else if (what == "replay") rc = run_replay(r, n, id);
      else if (what == "failure") rc = run_failure(r, n, id, dir, false);
      std::fflush(stdout);
      _exit(rc);
    }
    kids.push_back(p);
  }
  int bad = 0;
  if (what == "failure") {  // the replacement is spawned once the dying rank is gone
    int stt = 0;
    waitpid(kids.back(), &stt, 0);
    kids.pop_back();
    const pid_t p = fork();
    if (p == 0) {
      g_rank = n - 1;
      const int rc = run_failure(n - 1, n, id, dir, true);
      std::fflush(stdout);
      _exit(rc);
    }
    kids.push_back(p);
  }
  for (pid_t p : kids) {
    int st = 0;
    waitpid(p, &st, 0);
    if (!WIFEXITED(st) || WEXITSTATUS(st) != 0) ++bad;
  }
  std::printf("%s %s n=%d: %d process(es) failed\n", bad ? "FAIL" : "OK", what.c_str(), n, bad);
  return bad ? 1 : 0;
}

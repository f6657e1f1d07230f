// Copy-engine NVLink bandwidth with several concurrent peer flows (one
// process, 4 GPUs): does one GPU's outbound traffic to two or three peers
// exceed its single-peer copy-engine rate, and what does a balanced
// "two halves" broadcast pattern (every GPU sending to two peers, receiving
// the whole state) reach per receiver?
//   nvcc -O3 -std=c++17 tools/multipeer_bw.cu -o tools/multipeer_bw
//   ./tools/multipeer_bw [MiB per flow]
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CR(x)                                                                                   \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess) {                                                                    \
      std::printf("FAIL %s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_));  \
      std::exit(1);                                                                             \
    }                                                                                           \
  } while (0)

struct Flow {
  int src, dst;
  double frac;  // of the per-flow size
  int sm = 0;   // 1: SM stores from a kernel on src (peer mapping) instead of the copy engines
};

__global__ void __launch_bounds__(512) push_sm(const float4* __restrict__ src, float4* dst, size_t n16) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n16; i += size_t(gridDim.x) * blockDim.x)
    dst[i] = __ldg(src + i);
}

int ndev = 0;
size_t bytes = 0;
std::vector<char*> sbuf, dbuf;
std::vector<cudaStream_t> streams;  // one per (src, slot)

double run(const char* name, const std::vector<Flow>& flows, double recv_bytes) {
  // one stream per flow on its source device; start together behind an event on device 0
  std::vector<cudaStream_t> st(flows.size());
  for (size_t i = 0; i < flows.size(); ++i) {
    CR(cudaSetDevice(flows[i].src));
    CR(cudaStreamCreateWithFlags(&st[i], cudaStreamNonBlocking));
  }
  double best = 1e30;
  for (int rep = 0; rep < 6; ++rep) {
    for (int d = 0; d < ndev; ++d) {
      CR(cudaSetDevice(d));
      CR(cudaDeviceSynchronize());
    }
    // span on the host clock: all flows issued back to back (a few us), then every
    // device synchronised -- per-flow events would hide flows that serialise
    const auto t0 = std::chrono::steady_clock::now();
    for (size_t i = 0; i < flows.size(); ++i) {
      CR(cudaSetDevice(flows[i].src));
      const size_t n = size_t(bytes * flows[i].frac) & ~size_t(4095);
      // the i-th flow writes its own slice of the destination
      char* dp = dbuf[flows[i].dst] + (i % 4) * (bytes / 2);
      if (flows[i].sm) {
        push_sm<<<flows[i].sm, 512, 0, st[i]>>>(reinterpret_cast<const float4*>(sbuf[flows[i].src]),
                                                 reinterpret_cast<float4*>(dp), n / 16);
        CR(cudaGetLastError());
      } else {
        CR(cudaMemcpyPeerAsync(dp, flows[i].dst, sbuf[flows[i].src], flows[i].src, n, st[i]));
      }
    }
    for (size_t i = 0; i < flows.size(); ++i) CR(cudaStreamSynchronize(st[i]));
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (rep > 0 && ms < best) best = ms;
  }
  double out_gb = 0;
  for (auto& f : flows) out_gb += bytes * f.frac / 1e9;
  std::printf("%-44s %8.3f ms  total %6.2f GB -> %7.1f GB/s aggregate, %7.1f GB/s per receiver of %.2f GB\n", name,
              best, out_gb, out_gb / (best * 1e-3), recv_bytes / 1e9 / (best * 1e-3), recv_bytes / 1e9);
  for (size_t i = 0; i < flows.size(); ++i) {
    CR(cudaSetDevice(flows[i].src));
    cudaStreamDestroy(st[i]);
  }
  return best;
}

int main(int argc, char** argv) {
  CR(cudaGetDeviceCount(&ndev));
  bytes = (argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 2048ull) << 20;
  std::printf("devices %d, %.2f GB per flow unit\n", ndev, bytes / 1e9);
  sbuf.resize(ndev);
  dbuf.resize(ndev);
  for (int d = 0; d < ndev; ++d) {
    CR(cudaSetDevice(d));
    for (int p = 0; p < ndev; ++p)
      if (p != d) {
        int can = 0;
        CR(cudaDeviceCanAccessPeer(&can, d, p));
        if (can) cudaDeviceEnablePeerAccess(p, 0);
        cudaGetLastError();
      }
    CR(cudaMalloc(&sbuf[d], bytes));
    CR(cudaMalloc(&dbuf[d], 2 * bytes));
    CR(cudaMemset(sbuf[d], d + 1, bytes));
  }
  run("0->1", {{0, 1, 1.0}}, bytes);
  if (ndev >= 3) {
    run("0->1 + 0->2 (one GPU, two peers)", {{0, 1, 1.0}, {0, 2, 1.0}}, bytes);
    run("0->1 + 2->1 (two sources, one receiver)", {{0, 1, 0.5}, {2, 1, 0.5}}, bytes);
    run("0->1 + 1->2 (receive while sending)", {{0, 1, 1.0}, {1, 2, 1.0}}, bytes);
    run("0->1 x2 streams (one peer, two engines?)", {{0, 1, 0.5}, {0, 1, 0.5}}, bytes);
  }
  run("0->1 SM stores (296 CTAs)", {{0, 1, 1.0, 296}}, bytes);
  run("0->1 CE 0.5 + SM 0.5 (same peer)", {{0, 1, 0.5}, {0, 1, 0.5, 296}}, bytes);
  run("0->1 CE 0.55 + SM 0.45 (same peer, 74 CTAs)", {{0, 1, 0.55}, {0, 1, 0.45, 74}}, bytes);
  if (ndev >= 3) run("0->1 CE + 0->2 SM (two peers)", {{0, 1, 1.0}, {0, 2, 1.0, 296}}, bytes);
  if (ndev >= 4) {
    run("0->1 + 0->2 + 0->3", {{0, 1, 1.0}, {0, 2, 1.0}, {0, 3, 1.0}}, bytes);
    // halves: A = first half, B = second half of the state (bytes each = one half)
    run("halves: 0->{1:A,2:B} 1->{2,3}:A 2->{1,3}:B",
        {{0, 1, 0.5}, {0, 2, 0.5}, {1, 2, 0.5}, {1, 3, 0.5}, {2, 1, 0.5}, {2, 3, 0.5}}, bytes);
    run("chain 0->1->2->3 (all links at once)", {{0, 1, 1.0}, {1, 2, 1.0}, {2, 3, 1.0}}, bytes);
  }
  return 0;
}

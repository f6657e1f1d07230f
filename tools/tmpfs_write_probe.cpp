// Page-cache write rate of /dev/shm by thread count: write() from a private buffer
// (mode 0), memcpy into a MAP_SHARED mapping (mode 1), the same with MAP_POPULATE
// (mode 2).  g++ -O2 -pthread tools/tmpfs_write_probe.cpp -o tools/tmpfs_write_probe
//   ./tools/tmpfs_write_probe <threads> <MiB per thread> <mode>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>
int main(int argc, char** argv) {
  int nt = argc > 1 ? atoi(argv[1]) : 1;
  size_t per = (argc > 2 ? atol(argv[2]) : 256) << 20;
  int mode = argc > 3 ? atoi(argv[3]) : 0;
  std::vector<char*> src(nt);
  for (int i = 0; i < nt; ++i) { src[i] = (char*)aligned_alloc(4096, per); memset(src[i], i + 1, per); }
  auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> th;
  for (int i = 0; i < nt; ++i) th.emplace_back([&, i] {
    std::string p = "/dev/shm/wprobe_" + std::to_string(i);
    int fd = open(p.c_str(), O_CREAT | O_TRUNC | O_RDWR, 0644);
    if (mode == 0) {
      size_t off = 0;
      while (off < per) { ssize_t w = write(fd, src[i] + off, std::min(per - off, (size_t)64 << 20)); off += w; }
    } else {
      if (ftruncate(fd, per)) perror("ft");
      int fl = MAP_SHARED | (mode == 2 ? MAP_POPULATE : 0);
      char* m = (char*)mmap(nullptr, per, PROT_READ | PROT_WRITE, fl, fd, 0);
      memcpy(m, src[i], per);
      munmap(m, per);
    }
    close(fd);
  });
  for (auto& t : th) t.join();
  double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  printf("threads %d mode %d: %.2f GB/s\n", nt, mode, nt * per / s / 1e9);
  for (int i = 0; i < nt; ++i) unlink(("/dev/shm/wprobe_" + std::to_string(i)).c_str());
}

// HSDL v1 problem files (reference problem.cpp:144-243): header parsing shared by the
// drop-in and the engine's streaming loader (hsdl_file.cpp).
#pragma once

#include <unistd.h>

#include <cstdint>
#include <vector>

namespace hsdla_b200 {

struct HsdlHeader {
  uint64_t na = 0, nl = 0, ng = 0;
  uint64_t off_flags = 32, off_A = 0, off_B = 0, off_T = 0, off_U = 0, total = 0;
  std::vector<uint8_t> hpd;
};

struct Fd {
  int fd = -1;
  ~Fd() {
    if (fd >= 0) close(fd);
  }
};

// problem.cpp:197-225: magic "HSDL", version 1, dims, hpd bit flags; checked_total.
HsdlHeader read_hsdl_header(int fd, const char* path);
int open_hsdl(const char* path);

}  // namespace hsdla_b200

// Device-direct file I/O for the PPRG / PPRW formats: the file body streams
// through two pinned staging buffers straight into (or out of) device arrays,
// so a multi-GB graph never materialises as host vectors.
#pragma once
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdint>
#include <string>

#include "common.cuh"

namespace pprg {

struct FileCloser {
  FILE* f = nullptr;
  ~FileCloser() {
    if (f) std::fclose(f);
  }
};

class Staging {
 public:
  static constexpr size_t kChunk = 64ull << 20;
  explicit Staging(cudaStream_t st) : st_(st) {
    for (int i = 0; i < 2; ++i) {
      PPRG_CUDA(cudaHostAlloc(&buf_[i], kChunk, cudaHostAllocDefault));
      PPRG_CUDA(cudaEventCreateWithFlags(&ev_[i], cudaEventDisableTiming));
      PPRG_CUDA(cudaEventRecord(ev_[i], st_));
    }
  }
  ~Staging() {
    cudaStreamSynchronize(st_);
    for (int i = 0; i < 2; ++i) {
      cudaFreeHost(buf_[i]);
      cudaEventDestroy(ev_[i]);
    }
  }
  // file -> device, `bytes` at dst; false on a short read
  bool read(FILE* f, void* dst, size_t bytes) {
    char* d = static_cast<char*>(dst);
    for (size_t done = 0; done < bytes;) {
      const size_t len = bytes - done < kChunk ? bytes - done : kChunk;
      PPRG_CUDA(cudaEventSynchronize(ev_[slot_]));  // the slot's previous copy is done
      if (std::fread(buf_[slot_], 1, len, f) != len) return false;
      PPRG_CUDA(cudaMemcpyAsync(d + done, buf_[slot_], len, cudaMemcpyHostToDevice, st_));
      PPRG_CUDA(cudaEventRecord(ev_[slot_], st_));
      slot_ ^= 1;
      done += len;
    }
    return true;
  }
  // device -> file; false on a short write
  bool write(FILE* f, const void* src, size_t bytes) {
    const char* s = static_cast<const char*>(src);
    for (size_t done = 0; done < bytes;) {
      const size_t len = bytes - done < kChunk ? bytes - done : kChunk;
      PPRG_CUDA(cudaMemcpyAsync(buf_[0], s + done, len, cudaMemcpyDeviceToHost, st_));
      PPRG_CUDA(cudaStreamSynchronize(st_));
      if (std::fwrite(buf_[0], 1, len, f) != len) return false;
      done += len;
    }
    return true;
  }

 private:
  cudaStream_t st_;
  char* buf_[2] = {nullptr, nullptr};
  cudaEvent_t ev_[2] = {nullptr, nullptr};
  int slot_ = 0;
};

inline uint64_t file_size(FILE* f) {
  const long cur = std::ftell(f);
  std::fseek(f, 0, SEEK_END);
  const long end = std::ftell(f);
  std::fseek(f, cur, SEEK_SET);
  return end < 0 ? 0 : (uint64_t)end;
}

}  // namespace pprg

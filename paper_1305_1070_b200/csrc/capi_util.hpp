// Shared helpers of the C-ABI translation units (status mapping, CUDA
// checks, device uploads).
#pragma once

#include <cuda_runtime.h>

#include <cstdio>
#include <string>
#include <vector>

#include "negf_gpu.h"

namespace negfb {

inline int set_status(negf_status* st, int code, const std::string& msg, int energy = -1, int cluster = -1,
               int pivot = -1, int dof = -1) {
  if (st) {
    st->code = code;
    st->energy_index = energy;
    st->cluster = cluster;
    st->pivot = pivot;
    st->dof = dof;
    std::snprintf(st->msg, sizeof st->msg, "%s", msg.c_str());
  }
  return code;
}

inline int ok(negf_status* st) { return set_status(st, NEGF_OK, ""); }

struct CudaFail {
  int code;
  std::string msg;
};

inline void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    const int code = (e == cudaErrorMemoryAllocation) ? NEGF_OUT_OF_MEMORY : NEGF_CUDA_ERROR;
    throw CudaFail{code, std::string(what) + ": " + cudaGetErrorString(e)};
  }
}

template <class T>
inline T* dev_upload(const std::vector<T>& v, std::vector<void*>& owned) {
  if (v.empty()) return nullptr;
  T* p = nullptr;
  ck(cudaMalloc(&p, sizeof(T) * v.size()), "cudaMalloc");
  owned.push_back(p);
  ck(cudaMemcpy(p, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice), "upload");
  return p;
}

template <class T>
inline T* dev_alloc(size_t count, std::vector<void*>& owned) {
  if (count == 0) count = 1;
  T* p = nullptr;
  ck(cudaMalloc(&p, sizeof(T) * count), "cudaMalloc");
  owned.push_back(p);
  return p;
}

}  // namespace negfb

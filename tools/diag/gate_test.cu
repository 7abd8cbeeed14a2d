// Standalone check of cuStreamWaitValue32 on mapped pinned host memory (the
// pack-launch gate). Prints the outcome of each variant; every wait is bounded.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <chrono>
#include <cstdio>
#include <thread>

__global__ void k(int* x) { if (threadIdx.x == 0) atomicAdd(x, 1); }

static bool wait_done(cudaEvent_t e, double secs) {
  auto t0 = std::chrono::steady_clock::now();
  while (cudaEventQuery(e) == cudaErrorNotReady) {
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > secs) return false;
    std::this_thread::sleep_for(std::chrono::microseconds(100));
  }
  return true;
}

int main() {
  cudaSetDevice(0);
  int attr = -1;
  cuDeviceGetAttribute(&attr, CU_DEVICE_ATTRIBUTE_CAN_USE_STREAM_MEM_OPS_V1, 0);
  printf("CAN_USE_STREAM_MEM_OPS_V1=%d\n", attr);
  cuDeviceGetAttribute(&attr, CU_DEVICE_ATTRIBUTE_CAN_USE_HOST_POINTER_FOR_REGISTERED_MEM, 0);
  printf("CAN_USE_HOST_POINTER_FOR_REGISTERED_MEM=%d\n", attr);
  int* d; cudaMalloc(&d, 4);
  for (int variant = 0; variant < 4; ++variant) {
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaEvent_t e; cudaEventCreate(&e);
    volatile unsigned* h = nullptr; void* hp = nullptr;
    CUdeviceptr dp = 0;
    void* fn = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &fn, 11070, cudaEnableDefault, &q);
    auto wv = (PFN_cuStreamWaitValue32_v11070)fn;
    if (variant == 0) {          // cudaHostAlloc mapped, runtime entry point
      cudaHostAlloc(&hp, 4096, cudaHostAllocMapped | cudaHostAllocPortable);
      void* dv; cudaHostGetDevicePointer(&dv, hp, 0); dp = (CUdeviceptr)dv;
    } else if (variant == 1) {   // same memory, linked cuStreamWaitValue32
      cudaHostAlloc(&hp, 4096, cudaHostAllocMapped | cudaHostAllocPortable);
      void* dv; cudaHostGetDevicePointer(&dv, hp, 0); dp = (CUdeviceptr)dv;
      wv = (PFN_cuStreamWaitValue32_v11070)&cuStreamWaitValue32;
    } else if (variant == 2) {   // cuMemHostAlloc DEVICEMAP
      cuMemHostAlloc(&hp, 4096, CU_MEMHOSTALLOC_DEVICEMAP | CU_MEMHOSTALLOC_PORTABLE);
      cuMemHostGetDevicePointer(&dp, hp, 0);
    } else {                     // flush flag
      cudaHostAlloc(&hp, 4096, cudaHostAllocMapped | cudaHostAllocPortable);
      void* dv; cudaHostGetDevicePointer(&dv, hp, 0); dp = (CUdeviceptr)dv;
    }
    h = (volatile unsigned*)hp; *h = 0;
    unsigned flags = variant == 3 ? CU_STREAM_WAIT_VALUE_GEQ | CU_STREAM_WAIT_VALUE_FLUSH : CU_STREAM_WAIT_VALUE_GEQ;
    CUresult r = wv((CUstream)s, dp, 1, flags);
    k<<<1, 32, 0, s>>>(d);
    cudaEventRecord(e, s);
    std::this_thread::sleep_for(std::chrono::milliseconds(5));
    bool early = cudaEventQuery(e) == cudaSuccess;
    __atomic_store_n(h, 1u, __ATOMIC_SEQ_CST);
    bool ok = wait_done(e, 3.0);
    printf("variant %d: wait rc=%d entry=%d early=%d released=%d err=%s\n", variant, (int)r, (int)q,
           early, ok, cudaGetErrorString(cudaGetLastError()));
    fflush(stdout);
    if (!ok) { __atomic_store_n(h, 100u, __ATOMIC_SEQ_CST); wait_done(e, 2.0); }
  }
  return 0;
}

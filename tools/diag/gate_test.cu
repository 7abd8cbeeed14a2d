// Which host->GPU signalling works on this platform? Every wait is bounded;
// output is unbuffered (stderr) so a kill still leaves the trace.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <chrono>
#include <cstdio>
#include <thread>

__global__ void bump(int* x) { if (threadIdx.x == 0) atomicAdd(x, 1); }
__global__ void spin(const volatile unsigned* f, unsigned v, unsigned long long max_ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    unsigned x;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(x) : "l"(f));
    if ((int)(x - v) >= 0) return;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > max_ns) return;   // bounded
    __nanosleep(200);
  }
}

static bool wait_done(cudaEvent_t e, double secs) {
  auto t0 = std::chrono::steady_clock::now();
  while (cudaEventQuery(e) == cudaErrorNotReady) {
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > secs) return false;
    std::this_thread::sleep_for(std::chrono::microseconds(100));
  }
  return true;
}

int main(int argc, char** argv) {
  int which = argc > 1 ? atoi(argv[1]) : 0;
  cudaSetDevice(0);
  int a1 = -1, a2 = -1;
  cuDeviceGetAttribute(&a1, CU_DEVICE_ATTRIBUTE_CAN_USE_STREAM_MEM_OPS_V1, 0);
  cuDeviceGetAttribute(&a2, CU_DEVICE_ATTRIBUTE_CAN_USE_HOST_POINTER_FOR_REGISTERED_MEM, 0);
  fprintf(stderr, "mem_ops=%d host_ptr_reg=%d\n", a1, a2);
  int* d; cudaMalloc(&d, 4);
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e; cudaEventCreate(&e);
  void* hp = nullptr;
  cudaHostAlloc(&hp, 4096, cudaHostAllocMapped | cudaHostAllocPortable);
  void* dv; cudaHostGetDevicePointer(&dv, hp, 0);
  volatile unsigned* h = (volatile unsigned*)hp; *h = 0;
  if (which == 0) {   // spin kernel on the mapped flag
    spin<<<1, 32, 0, s>>>((const volatile unsigned*)dv, 1, 3000000000ull);
    bump<<<1, 32, 0, s>>>(d);
    cudaEventRecord(e, s);
    std::this_thread::sleep_for(std::chrono::milliseconds(20));
    bool early = cudaEventQuery(e) == cudaSuccess;
    auto t0 = std::chrono::steady_clock::now();
    __atomic_store_n(h, 1u, __ATOMIC_SEQ_CST);
    bool ok = wait_done(e, 5.0);
    double dt = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    fprintf(stderr, "spin: early=%d released=%d after %.6f s err=%s\n", early, ok, dt,
            cudaGetErrorString(cudaGetLastError()));
  } else {            // cuStreamWaitValue32 on device memory, released by cuStreamWriteValue32
    unsigned* dflag; cudaMalloc(&dflag, 4); cudaMemset(dflag, 0, 4); cudaDeviceSynchronize();
    cudaStream_t s2; cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    CUresult r = cuStreamWaitValue32((CUstream)s, (CUdeviceptr)dflag, 1, CU_STREAM_WAIT_VALUE_GEQ);
    fprintf(stderr, "waitvalue(dev) rc=%d\n", (int)r);
    bump<<<1, 32, 0, s>>>(d);
    cudaEventRecord(e, s);
    std::this_thread::sleep_for(std::chrono::milliseconds(20));
    bool early = cudaEventQuery(e) == cudaSuccess;
    r = cuStreamWriteValue32((CUstream)s2, (CUdeviceptr)dflag, 1, 0);
    fprintf(stderr, "writevalue rc=%d\n", (int)r);
    bool ok = wait_done(e, 5.0);
    fprintf(stderr, "waitvalue(dev): early=%d released=%d err=%s\n", early, ok,
            cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}

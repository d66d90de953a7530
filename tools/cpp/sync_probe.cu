// Which CUDA runtime calls block the calling host thread while ANOTHER stream of the same
// device holds a kernel spinning on a flag that only later work will set?  (Ranks sharing one
// GPU in the peer-memory tests: a call that waits for the whole device deadlocks there.)
// Each probe: stream A runs a spinner (1 CTA) that exits when *flag != 0 or after 3 s; the host
// times the call under test on stream B, then releases the spinner.
//   make -C tools/cpp sync_probe && tools/cpp/sync_probe
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <functional>

__global__ void spin(volatile int* flag, unsigned long long ns) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    if (*flag) return;
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > ns) return;
    __nanosleep(200);
  }
}

int main() {
  int* flag;
  cudaMalloc(&flag, 4);
  cudaStream_t a, b;
  cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
  void* keep = nullptr;
  cudaMalloc(&keep, 1 << 20);
  auto probe = [&](const char* name, const std::function<void()>& f) {
    cudaMemset(flag, 0, 4);
    cudaDeviceSynchronize();
    spin<<<1, 32, 0, a>>>(flag, 3000000000ull);
    cudaStreamQuery(a);
    auto t0 = std::chrono::steady_clock::now();
    f();
    double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    int one = 1;
    cudaMemcpyAsync(flag, &one, 4, cudaMemcpyHostToDevice, b);
    cudaDeviceSynchronize();
    printf("{\"call\": \"%s\", \"host_ms\": %.2f, \"blocks_on_other_stream\": %s}\n", name, ms,
           ms > 1000 ? "true" : "false");
  };
  void* p = nullptr;
  probe("cudaMalloc 64MB", [&] { cudaMalloc(&p, 64 << 20); });
  probe("cudaFree", [&] { cudaFree(p); });
  probe("cudaMallocAsync 64MB (fresh pool)", [&] { cudaMallocAsync(&p, 64 << 20, b); });
  probe("cudaFreeAsync", [&] { cudaFreeAsync(p, b); });
  probe("cudaMallocAsync 256MB (pool growth)", [&] { cudaMallocAsync(&p, 256 << 20, b); });
  probe("cudaMemsetAsync", [&] { cudaMemsetAsync(p, 0, 1 << 20, b); });
  probe("cudaFreeAsync 2", [&] { cudaFreeAsync(p, b); });
  probe("cudaStreamSynchronize(b)", [&] { cudaStreamSynchronize(b); });
  probe("cudaMemset (legacy)", [&] { cudaMemset(keep, 0, 1 << 20); });
  probe("cudaMemcpy D2H (legacy)", [&] { int h; cudaMemcpy(&h, keep, 4, cudaMemcpyDeviceToHost); });
  probe("cudaHostAlloc", [&] { void* h; cudaHostAlloc(&h, 1 << 20, 0); });
  probe("cudaEventCreate", [&] { cudaEvent_t e; cudaEventCreate(&e); });
  probe("cudaStreamCreate", [&] { cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking); });
  probe("cudaStreamDestroy", [&] { cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking); cudaStreamDestroy(s); });
  probe("cudaDeviceSynchronize", [&] { cudaDeviceSynchronize(); });
  return 0;
}

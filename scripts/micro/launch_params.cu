// Launch-latency microbenchmark: event -> one kernel with a P-byte parameter block -> event,
// after a spin gate so the host has enqueued everything; and the same for a PDL-chained pair.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lp launch_params.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int P> struct Blob { unsigned char b[P]; };

__global__ void spin(long long cycles) {
  long long t0 = clock64();
  while (clock64() - t0 < cycles) {}
}
template <int P> __global__ void k(Blob<P> a, int* out) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (threadIdx.x == 0 && a.b[P - 1] == 7) out[0] = 1;
}

template <int P> float measure(cudaStream_t s, int* d, int nk, bool pdl) {
  Blob<P> a{};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e9;
  for (int rep = 0; rep < 50; ++rep) {
    spin<<<1, 1, 0, s>>>(2000000);
    cudaEventRecord(e0, s);
    for (int i = 0; i < nk; ++i) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(1); cfg.blockDim = dim3(256); cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at; cfg.numAttrs = pdl ? 1 : 0;
      cudaLaunchKernelEx(&cfg, k<P>, a, d);
    }
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 5 && ms < best) best = ms;
  }
  return best * 1e3f;
}

int main() {
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  int* d; cudaMalloc(&d, 4);
  for (int pdl = 0; pdl < 2; ++pdl)
    for (int nk : {1, 2, 6}) {
      printf("pdl=%d kernels=%d: P=64 %.2f us  P=1024 %.2f us  P=4096 %.2f us\n", pdl, nk,
             measure<64>(s, d, nk, pdl), measure<1024>(s, d, nk, pdl), measure<4096>(s, d, nk, pdl));
    }
  return 0;
}

// Minimal TMA load test: 1D float64 box / 2D float32 rows into shared memory, tensor map in
// kernel parameter space (grid constant) or in global memory.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include "../../paper_2404_16221_b200/csrc/tma.cuh"

struct Maps { CUtensorMap a, v; };

__global__ void k(const __grid_constant__ Maps m, const Maps* gm, double* out, int mode) {
  __shared__ __align__(128) double buf[128];
  __shared__ __align__(128) float vb[512];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) { vr::tma::mbar_init(&bar, 1); vr::tma::fence_init(); }
  __syncthreads();
  const Maps* mp = (mode & 2) ? gm : &m;
  if (threadIdx.x == 0) {
    if (mode & 1) {
      vr::tma::expect_tx(&bar, 2048);
      vr::tma::load_2d(vb, &mp->v, 0, 5, &bar);
    } else {
      vr::tma::expect_tx(&bar, 1024);
      vr::tma::load_1d(buf, &mp->a, 10, &bar);
    }
  }
  vr::tma::wait(&bar, 0);
  out[threadIdx.x] = (mode & 1) ? vb[4 * threadIdx.x] : buf[threadIdx.x];
}

int main(int argc, char** argv) {
  int mode = argc > 1 ? atoi(argv[1]) : 0;
  double *d, *o; float* f; Maps* gm;
  cudaMalloc(&d, 8 * 1024); cudaMalloc(&o, 8 * 128); cudaMalloc(&f, 16 * 1024);
  cudaMalloc(&gm, sizeof(Maps));
  double h[1024]; for (int i = 0; i < 1024; ++i) h[i] = i;
  float hf[4096]; for (int i = 0; i < 4096; ++i) hf[i] = 1000 + i;
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaMemcpy(f, hf, sizeof(hf), cudaMemcpyHostToDevice);
  Maps m;
  bool ok1 = vr::tma::encode_1d(&m.a, d, 1024, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, 128);
  bool ok2 = vr::tma::encode_rows(&m.v, f, 1024, 4, 128);
  cudaMemcpy(gm, &m, sizeof(m), cudaMemcpyHostToDevice);
  printf("encode %d %d sizeof(Maps) %zu\n", ok1, ok2, sizeof(Maps));
  k<<<1, 128>>>(m, gm, o, mode);
  cudaError_t e = cudaDeviceSynchronize();
  double ho[128]; cudaMemcpy(ho, o, sizeof(ho), cudaMemcpyDeviceToHost);
  printf("mode %d: %s  out[0]=%g out[1]=%g\n", mode, cudaGetErrorString(e), ho[0], ho[1]);
  return e != cudaSuccess;
}

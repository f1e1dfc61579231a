#include <cstdio>
#include <cmath>
// m16n8k4 f64 fragment-layout check: A 16x4, B 4x8, D = A B
__global__ void k(const double* A, const double* B, double* D) {
  const int l = threadIdx.x, g = l / 4, t = l % 4;
  double a0 = A[g * 4 + t], a1 = A[(g + 8) * 4 + t], b0 = B[t * 8 + g];
  double d0 = 0, d1 = 0, d2 = 0, d3 = 0;
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(d0), "+d"(d1), "+d"(d2), "+d"(d3) : "d"(a0), "d"(a1), "d"(b0));
  D[g * 8 + 2 * t] = d0; D[g * 8 + 2 * t + 1] = d1; D[(g + 8) * 8 + 2 * t] = d2; D[(g + 8) * 8 + 2 * t + 1] = d3;
}
int main() {
  double hA[64], hB[32], hD[128], R[128];
  for (int i = 0; i < 64; ++i) hA[i] = (i * 7 % 13) - 6;
  for (int i = 0; i < 32; ++i) hB[i] = (i * 5 % 11) - 5;
  for (int r = 0; r < 16; ++r) for (int c = 0; c < 8; ++c) { double s = 0; for (int k = 0; k < 4; ++k) s += hA[r * 4 + k] * hB[k * 8 + c]; R[r * 8 + c] = s; }
  double *dA, *dB, *dD; cudaMalloc(&dA, 512); cudaMalloc(&dB, 256); cudaMalloc(&dD, 1024);
  cudaMemcpy(dA, hA, 512, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice);
  k<<<1, 32>>>(dA, dB, dD); cudaMemcpy(hD, dD, 1024, cudaMemcpyDeviceToHost);
  double err = 0; for (int i = 0; i < 128; ++i) err = fmax(err, fabs(hD[i] - R[i]));
  printf("m16n8k4 layout max err %g (%s)\n", err, cudaGetErrorString(cudaGetLastError()));
}

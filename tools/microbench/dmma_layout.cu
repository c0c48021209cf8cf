// Fragment layouts of the sm_90+ FP64 mma.sync shapes m16n8k8 / m16n8k16 on
// sm_100a, checked against a CPU product (g = lane>>2, t = lane&3):
//   A (16 x K, row): a_i = A[g + 8*(i%2)][t + 4*(i/2)]
//   B (K x 8, col):  b_i = B[t + 4*i][g]
//   C (16 x 8):      c0,c1 = C[g][2t], C[g][2t+1];  c2,c3 = C[g+8][2t], C[g+8][2t+1]
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench/dmma_layout tools/microbench/dmma_layout.cu
#include <cstdio>
#include <cmath>

template <int K>
__global__ void mma_once(const double* A, const double* B, double* C) {
  const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
  double a[K / 2], b[K / 4], c[4] = {0, 0, 0, 0};
#pragma unroll
  for (int i = 0; i < K / 2; ++i) a[i] = A[(g + 8 * (i % 2)) * K + t + 4 * (i / 2)];
#pragma unroll
  for (int i = 0; i < K / 4; ++i) b[i] = B[(t + 4 * i) * 8 + g];
  if (K == 8)
    asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(b[0]), "d"(b[1]));
  else
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};\n"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                 : "d"(a[0]), "d"(a[1]), "d"(a[2 % (K / 2)]), "d"(a[3 % (K / 2)]), "d"(a[4 % (K / 2)]), "d"(a[5 % (K / 2)]),
                   "d"(a[6 % (K / 2)]), "d"(a[7 % (K / 2)]), "d"(b[0]), "d"(b[1]), "d"(b[2 % (K / 4)]), "d"(b[3 % (K / 4)]));
  C[g * 8 + 2 * t] = c[0]; C[g * 8 + 2 * t + 1] = c[1];
  C[(g + 8) * 8 + 2 * t] = c[2]; C[(g + 8) * 8 + 2 * t + 1] = c[3];
}

template <int K>
int check() {
  double hA[16 * K], hB[K * 8], hC[128], ref[128];
  for (int i = 0; i < 16 * K; ++i) hA[i] = std::sin(1.0 + 0.37 * i);
  for (int i = 0; i < K * 8; ++i) hB[i] = std::cos(0.5 + 0.23 * i);
  for (int m = 0; m < 16; ++m)
    for (int n = 0; n < 8; ++n) {
      double s = 0; for (int k = 0; k < K; ++k) s += hA[m * K + k] * hB[k * 8 + n];
      ref[m * 8 + n] = s;
    }
  double *A, *B, *C;
  cudaMalloc(&A, sizeof(hA)); cudaMalloc(&B, sizeof(hB)); cudaMalloc(&C, sizeof(hC));
  cudaMemcpy(A, hA, sizeof(hA), cudaMemcpyHostToDevice); cudaMemcpy(B, hB, sizeof(hB), cudaMemcpyHostToDevice);
  mma_once<K><<<1, 32>>>(A, B, C);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(hC, C, sizeof(hC), cudaMemcpyDeviceToHost);
  double err = 0; for (int i = 0; i < 128; ++i) err = std::fmax(err, std::fabs(hC[i] - ref[i]));
  printf("m16n8k%-2d max |C - ref| = %.3e  (%s)\n", K, err, cudaGetErrorString(e));
  return err < 1e-12 ? 0 : 1;
}

int main() { return check<8>() | check<16>(); }

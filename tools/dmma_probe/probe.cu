// Probe of the mma.sync m16n8k4 f64 fragment layout (run on a B200):
// D = A (16x4, row) * B (4x8, col) with the assumed layout, compared with
// a host reference.  Prints max abs error.
#include <cstdio>
#include <cmath>
__global__ void k(const double *A, const double *B, double *D) {
    const int lane = threadIdx.x, gid = lane >> 2, tig = lane & 3;
    double a0 = A[gid * 4 + tig], a1 = A[(gid + 8) * 4 + tig];
    double b0 = B[tig * 8 + gid];  // B[k][n]
    double c0 = 0, c1 = 0, c2 = 0, c3 = 0;
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                 : "+d"(c0), "+d"(c1), "+d"(c2), "+d"(c3) : "d"(a0), "d"(a1), "d"(b0));
    D[gid * 8 + 2 * tig] = c0;
    D[gid * 8 + 2 * tig + 1] = c1;
    D[(gid + 8) * 8 + 2 * tig] = c2;
    D[(gid + 8) * 8 + 2 * tig + 1] = c3;
}
int main() {
    double hA[64], hB[32], hD[128], ref[128];
    for (int i = 0; i < 64; ++i) hA[i] = (i * 7 % 13) - 6;
    for (int i = 0; i < 32; ++i) hB[i] = (i * 5 % 11) - 5;
    for (int r = 0; r < 16; ++r)
        for (int c = 0; c < 8; ++c) {
            double s = 0;
            for (int q = 0; q < 4; ++q) s += hA[r * 4 + q] * hB[q * 8 + c];
            ref[r * 8 + c] = s;
        }
    double *dA, *dB, *dD;
    cudaMalloc(&dA, sizeof hA); cudaMalloc(&dB, sizeof hB); cudaMalloc(&dD, sizeof hD);
    cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
    k<<<1, 32>>>(dA, dB, dD);
    cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
    double e = 0;
    for (int i = 0; i < 128; ++i) e = fmax(e, fabs(hD[i] - ref[i]));
    printf("dmma m16n8k4 f64 layout max err %g\n", e);
    return 0;
}

// Dependent-DADD latency probe: one thread runs a chain of N dependent adds.
// Build + run on the GPU box: nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/dadd tools/probes/dadd_latency.cu && /tmp/dadd
#include <cstdio>
__global__ void chain(double *out, double v, long long n, long long *cyc) {
    double a = 0.0, b = 1.0;
    long long t0 = clock64();
    for (long long i = 0; i < n; ++i) { a = __dadd_rn(a, v); b = __dadd_rn(b, v); }
    long long t1 = clock64();
    out[0] = a + b;
    *cyc = t1 - t0;
}
int main() {
    double *o; long long *c, h;
    cudaMalloc(&o, 8); cudaMalloc(&c, 8);
    const long long n = 1 << 20;
    chain<<<1, 1>>>(o, 1e-3, n, c);
    chain<<<1, 1>>>(o, 1e-3, n, c);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("dependent DADD: %.2f cycles per add (2 interleaved chains)\n", double(h) / n);
    return 0;
}

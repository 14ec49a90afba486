// Dependent-chain latency and throughput of the FP64 ops the RT3D path uses
// (compiled like librt3d: -fmad=false).
#include <cstdio>
#include <cmath>
template <int OP>
__global__ void chain(double* out, int iters, double a) {
    double x = a + threadIdx.x * 1e-9, y = 1.0000001;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (OP == 0) x = x + y;
        if (OP == 1) x = x * y;
        if (OP == 2) x = x / 1.0000003;
        if (OP == 3) x = sqrt(x) + 1.0;
        if (OP == 4) x = log(x) + 2.0;
        if (OP == 5) x = (double)(long long)(x) + 1.5;   // cvt
        if (OP == 6) x = floor(x) + 1.25;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (double)(t1 - t0) / iters;
    out[1 + threadIdx.x + blockIdx.x * blockDim.x] = x;
}
int main() {
    double* d;
    cudaMalloc(&d, 8 * (1 + 148 * 1024 * 2));
    const char* names[] = {"dadd", "dmul", "ddiv", "dsqrt+add", "log+add", "cvt ll->d", "floor+add"};
    for (int op = 0; op < 7; ++op) {
        double h;
        auto run = [&](int blocks, int threads) {
            cudaEvent_t a, b;
            cudaEventCreate(&a); cudaEventCreate(&b);
            int it = 4096;
            cudaEventRecord(a);
            switch (op) {
                case 0: chain<0><<<blocks, threads>>>(d, it, 1.5); break;
                case 1: chain<1><<<blocks, threads>>>(d, it, 1.5); break;
                case 2: chain<2><<<blocks, threads>>>(d, it, 1.5); break;
                case 3: chain<3><<<blocks, threads>>>(d, it, 1.5); break;
                case 4: chain<4><<<blocks, threads>>>(d, it, 1.5); break;
                case 5: chain<5><<<blocks, threads>>>(d, it, 1.5); break;
                case 6: chain<6><<<blocks, threads>>>(d, it, 1.5); break;
            }
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            double ops = (double)blocks * threads * it;
            return std::pair<double,double>(h, ops / (ms * 1e-3) / 1e12);
        };
        auto lat = run(1, 32);
        auto thr = run(148 * 8, 256);
        printf("%-10s latency %.1f cyc/op (1 warp)   throughput %.2f Top/s (148x8x256 threads)\n", names[op], lat.first, thr.second);
    }
}

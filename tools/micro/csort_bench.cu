// Phase timing of k_csort (globaltimer stamps, CTA 0) on a synthetic ready set:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -DCS_TIMING \
//        tools/micro/csort_bench.cu -o tools/micro/csort_bench
#include "../../paper_2411_03519_b200/csrc/am_sort.cu"
#include <cstdio>
#include <vector>
using namespace am;

int main(int argc, char** argv)
{
    int maxsm = 0;
    cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
    cudaFuncSetAttribute(k_csort, cudaFuncAttributeMaxDynamicSharedMemorySize, maxsm);
    cudaFuncSetAttribute(k_csort, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int n : {100, 42000}) {
        Dev d{};
        Ctl* ctl;
        cudaMalloc(&ctl, sizeof(Ctl));
        Ctl h{};
        h.n_ready = n;
        h.sort_bits = 27;
        cudaMemcpy(ctl, &h, sizeof h, cudaMemcpyHostToDevice);
        d.ctl = ctl;
        std::vector<unsigned long long> k(n);
        std::vector<uint32_t> v(n);
        for (int i = 0; i < n; i++) { k[i] = ((unsigned long long)(i * 7919 % 80) << 20) | (i * 13 % n); v[i] = i; }
        for (int j = 0; j < 2; j++) {
            cudaMalloc(&d.rkey[j], 8 * (size_t)n); cudaMalloc(&d.rval[j], 4 * (size_t)n);
        }
        unsigned long long kor = 0;
        for (int i = 0; i < n; i++) kor |= k[i];
        h.sort_or = kor;   // k_csort derives the pass count from the OR of the keys
        cudaMemcpy(ctl, &h, sizeof h, cudaMemcpyHostToDevice);
        cudaMemcpy(d.rkey[0], k.data(), 8 * (size_t)n, cudaMemcpyHostToDevice);
        cudaMemcpy(d.rval[0], v.data(), 4 * (size_t)n, cudaMemcpyHostToDevice);
        int32_t* order;
        cudaMalloc(&order, 4 * (size_t)n);
        cudaLaunchConfig_t lc{};
        lc.gridDim = dim3(16);
        lc.blockDim = dim3(1024);
        lc.dynamicSmemBytes = maxsm;
        cudaLaunchAttribute at{};
        at.id = cudaLaunchAttributeClusterDimension;
        at.val.clusterDim.x = 16; at.val.clusterDim.y = 1; at.val.clusterDim.z = 1;
        lc.attrs = &at; lc.numAttrs = 1;
        for (int rep = 0; rep < 3; rep++) {
            // the passes reuse rkey[0] as a ping-pong buffer: restore the input
            cudaMemcpy(d.rkey[0], k.data(), 8 * (size_t)n, cudaMemcpyHostToDevice);
            cudaEvent_t a, b;
            cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a);
            cudaLaunchKernelEx(&lc, k_csort, d, order, maxsm);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            unsigned long long t[128];
            cudaMemcpyFromSymbol(t, g_cs_t, sizeof t);
            printf("n=%d rep %d: %.2f us total (%s); stamps (us from start):", n, rep, ms * 1000,
                   cudaGetErrorString(cudaGetLastError()));
            for (int q = 1; q < 32; q++) if (t[q] >= t[0] && t[q] - t[0] < 1000000) printf(" %d:%.2f", q, (t[q] - t[0]) / 1000.0);
            printf("\n");
            cudaMemset(g_cs_t, 0, 0);
        }
        std::vector<int32_t> o(n);
        cudaMemcpy(o.data(), order, 4 * (size_t)n, cudaMemcpyDeviceToHost);
        bool ok = true;
        for (int i = 1; i < n; i++) {
            unsigned long long a = k[o[i - 1]], b = k[o[i]];
            if (a > b || (a == b && o[i - 1] > o[i])) { ok = false; break; }
        }
        printf("n=%d sorted=%d\n", n, ok);
    }
    return 0;
}

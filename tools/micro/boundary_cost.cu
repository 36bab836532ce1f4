// Calibration for DESIGN section 11 item 5: what does one dependent grid-wide step cost
// on this B200 when it is (a) a separate kernel launched with programmatic dependent
// launch (PDL) inside a CUDA graph, (b) a separate kernel without PDL, (c) a grid
// barrier inside one persistent cooperative kernel (cooperative_groups grid.sync), and
// (d) a hand-rolled sense-reversing grid barrier (one atomic per CTA)?  Each step does a
// trivial coalesced 1M-element pass so the CTAs are real; 12 steps per chain (the replay
// round's main stream), timed with events over 200 graph replays.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/micro/boundary_cost.cu -o tools/micro/boundary_cost
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>

namespace cg = cooperative_groups;

constexpr int kSteps = 12;
constexpr int kN = 1 << 20;

__device__ __forceinline__ void pass(uint32_t* a, int step)
{
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < kN; i += gridDim.x * blockDim.x) a[i] += (uint32_t)step;
}

__global__ void k_step(uint32_t* a, int step, int pdl)
{
    if (pdl) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        asm volatile("griddepcontrol.launch_dependents;");
    }
    pass(a, step);
}

__global__ void k_coop(uint32_t* a)
{
    cg::grid_group g = cg::this_grid();
    for (int s = 0; s < kSteps; s++) {
        pass(a, s);
        g.sync();
    }
}

// sense-reversing barrier: one arrival atomic per CTA, the last flips the generation
__device__ __forceinline__ void grid_barrier(unsigned* count, volatile unsigned* gen, unsigned nblocks)
{
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g0 = *gen;
        __threadfence();
        if (atomicAdd(count, 1u) == nblocks - 1) {
            *count = 0;
            __threadfence();
            *gen = g0 + 1;
        } else {
            while (*gen == g0) {}
        }
        __threadfence();
    }
    __syncthreads();
}

__global__ void k_persist(uint32_t* a, unsigned* count, unsigned* gen)
{
    for (int s = 0; s < kSteps; s++) {
        pass(a, s);
        grid_barrier(count, gen, gridDim.x);
    }
}

static cudaError_t launch_step(cudaStream_t st, int grid, uint32_t* a, int s, int pdl)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = 256;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k_step, a, s, pdl);
}

int main()
{
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_coop, 256, 0);
    const int grid = sms * (per_sm < 4 ? per_sm : 4);
    uint32_t* a;
    unsigned* bar;
    cudaMalloc(&a, 4 * kN);
    cudaMalloc(&bar, 8);
    cudaMemset(a, 0, 4 * kN);
    cudaMemset(bar, 0, 8);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int reps = 200;
    auto time_graph = [&](auto enqueue, const char* name) {
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
        enqueue();
        cudaStreamEndCapture(st, &g);
        if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("%s: instantiate failed\n", name); return; }
        for (int k = 0; k < 10; k++) cudaGraphLaunch(ge, st);
        cudaEventRecord(e0, st);
        for (int k = 0; k < reps; k++) cudaGraphLaunch(ge, st);
        cudaEventRecord(e1, st);
        cudaStreamSynchronize(st);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const cudaError_t e = cudaGetLastError();
        printf("{\"variant\": \"%s\", \"grid\": %d, \"steps\": %d, \"us_per_chain\": %.2f, \"us_per_step\": %.2f, \"err\": \"%s\"}\n",
               name, grid, kSteps, 1000.0 * ms / reps, 1000.0 * ms / reps / kSteps, cudaGetErrorString(e));
        cudaGraphExecDestroy(ge);
        cudaGraphDestroy(g);
    };
    time_graph([&] { for (int s = 0; s < kSteps; s++) launch_step(st, grid, a, s, 1); }, "kernels_pdl");
    time_graph([&] { for (int s = 0; s < kSteps; s++) launch_step(st, grid, a, s, 0); }, "kernels_plain");
    time_graph([&] {
        void* args[] = {&a};
        cudaLaunchCooperativeKernel((void*)k_coop, grid, 256, args, 0, st);
    }, "coop_grid_sync");
    time_graph([&] { k_persist<<<grid, 256, 0, st>>>(a, bar, bar + 1); }, "persistent_own_barrier");
    // one step alone: the floor of a single pass (launch included)
    time_graph([&] { launch_step(st, grid, a, 0, 0); }, "single_step");
    return 0;
}

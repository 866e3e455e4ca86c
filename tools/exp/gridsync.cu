// Feasibility probe: cost of a cooperative grid-wide sync on B200 at pass A's grid (592 x 128),
// whether a cooperative launch combines with programmatic stream serialisation, and whether it
// can be captured into a CUDA graph.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gridsync gridsync.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__global__ void work(float *buf, int n, int sync)
{
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n)
        buf[i] = buf[i] * 0.5f + 1.0f;
    if (sync)
        cg::this_grid().sync();
    if (i < n)
        buf[(i + 4096) % n] += 1.0f;
}

static float run(int grid, int sync, int coop, int pdl, int graph, int reps)
{
    float *buf;
    cudaMalloc(&buf, sizeof(float) * grid * 128);
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    int n = grid * 128;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (coop) {
        attr[na].id = cudaLaunchAttributeCooperative;
        attr[na].val.cooperative = 1;
        ++na;
    }
    if (pdl) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(128);
    cfg.stream = s;
    cfg.attrs = attr;
    cfg.numAttrs = na;
    cudaGraphExec_t ge = nullptr;
    if (graph) {
        cudaGraph_t g;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        for (int r = 0; r < reps; ++r)
            cudaLaunchKernelEx(&cfg, work, buf, n, sync);
        cudaError_t e = cudaStreamEndCapture(s, &g);
        if (e != cudaSuccess) {
            printf("capture failed: %s\n", cudaGetErrorString(e));
            return -1;
        }
        e = cudaGraphInstantiate(&ge, g, 0);
        if (e != cudaSuccess) {
            printf("instantiate failed: %s\n", cudaGetErrorString(e));
            return -1;
        }
    }
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 2; ++w) {
        cudaEventRecord(a, s);
        if (graph)
            cudaGraphLaunch(ge, s);
        else
            for (int r = 0; r < reps; ++r)
                cudaLaunchKernelEx(&cfg, work, buf, n, sync);
        cudaEventRecord(b, s);
        cudaStreamSynchronize(s);
    }
    cudaError_t e = cudaGetLastError();
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (e != cudaSuccess)
        printf("error: %s\n", cudaGetErrorString(e));
    cudaFree(buf);
    return ms * 1000.0f / reps;
}

int main()
{
    const int reps = 200;
    for (int grid : {148, 592}) {
        printf("grid %d: plain %.2f us, sync(coop) %.2f us, coop no sync %.2f us\n", grid, run(grid, 0, 0, 0, 0, reps),
               run(grid, 1, 1, 0, 0, reps), run(grid, 0, 1, 0, 0, reps));
        printf("grid %d: pdl plain %.2f us, pdl+coop+sync %.2f us\n", grid, run(grid, 0, 0, 1, 0, reps),
               run(grid, 1, 1, 1, 0, reps));
        printf("grid %d: graph pdl plain %.2f us, graph pdl+coop+sync %.2f us, graph coop+sync %.2f us\n", grid,
               run(grid, 0, 0, 1, 1, reps), run(grid, 1, 1, 1, 1, reps), run(grid, 1, 1, 0, 1, reps));
    }
    return 0;
}

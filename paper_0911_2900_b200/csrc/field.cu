// field.cu -- the static floor field on the device, bit-identical to compute_static_field.
//
// Reference: compute_static_field (world.hpp:220-266): multi-source Dijkstra from every Exit,
// 8-neighbour steps of 1 and sqrt(2) (fp64 adds), Walls skipped, a diagonal blocked when both
// orthogonal cells are Wall (world.hpp:212-216), periodic wrap in x.
//
// Device algorithm: Dial's buckets of width 1.  Every edge weighs >= 1 and fp64 rounding is
// monotone, so a cell whose value lies in [k, k+1) can only be improved from buckets < k; after
// buckets 0..k-1 have been relaxed, bucket k is final and can be relaxed in parallel.  The value
// stored is the minimum over walks of the left-folded fp64 sums, which is exactly what the
// reference's Dijkstra produces (tie order does not change values).  Relaxation uses a 64-bit
// atomicMin on the IEEE bits (non-negative doubles order like their bit patterns).
// Three rolling frontier lists (k, k+1, k+2) hold the cells to relax.
#include <math.h>

#include "internal.cuh"

struct FieldArgs {
    int W, H, boundary;
    const uint8_t* cells;
    unsigned long long* s;     // fp64 bits
    uint32_t* lists[3];
    unsigned int* counts;      // [3]
    int* inq;                  // bucket+1 the cell was last queued in
};

__global__ void field_init_kernel(FieldArgs a, size_t n) {
    FP_PDL_WAIT();
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const bool ex = a.cells[i] == FP_CELL_EXIT;
        a.s[i] = ex ? 0ull : 0x7ff0000000000000ull;
        a.inq[i] = ex ? 1 : 0;
        if (ex) {
            const unsigned slot = atomicAdd(&a.counts[0], 1u);
            a.lists[0][slot] = (uint32_t)i;
        }
    }
}

__device__ __forceinline__ int wrapx(const FieldArgs& a, int x) {
    if (a.boundary == FP_BOUNDARY_PERIODIC_X) {
        x %= a.W;
        if (x < 0) x += a.W;
    }
    return x;
}

__global__ void field_relax_kernel(FieldArgs a, int k) {
    FP_PDL_WAIT();
    const int cur = k % 3;
    const unsigned cnt = a.counts[cur];
    const uint32_t* list = a.lists[cur];
    const double diag = 0x1.6a09e667f3bcdp+0;  // sqrt(2.0), correctly rounded
    for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < cnt; t += gridDim.x * blockDim.x) {
        const uint32_t idx = list[t];
        const double d = __longlong_as_double((long long)a.s[idx]);
        if ((int)floor(d) != k) continue;  // stale entry: relaxed from an earlier bucket
        const int cx = (int)(idx % (uint32_t)a.W), cy = (int)(idx / (uint32_t)a.W);
        #pragma unroll
        for (int o = 0; o < 8; ++o) {
            const int ox = (o < 3) ? o - 1 : (o == 3 ? -1 : (o == 4 ? 1 : o - 6));
            const int oy = (o < 3) ? -1 : (o < 5 ? 0 : 1);
            const int ny = cy + oy;
            if (ny < 0 || ny >= a.H) continue;
            int nx = cx + ox;
            if (a.boundary == FP_BOUNDARY_PERIODIC_X) nx = wrapx(a, nx);
            else if (nx < 0 || nx >= a.W) continue;
            const size_t ni = (size_t)ny * a.W + nx;
            if (a.cells[ni] == FP_CELL_WALL) continue;
            if (ox != 0 && oy != 0) {
                const int sax = wrapx(a, cx + ox);
                if (a.cells[(size_t)cy * a.W + sax] == FP_CELL_WALL &&
                    a.cells[(size_t)ny * a.W + cx] == FP_CELL_WALL)
                    continue;
            }
            const double nd = __dadd_rn(d, (ox != 0 && oy != 0) ? diag : 1.0);
            const unsigned long long nb = (unsigned long long)__double_as_longlong(nd);
            const unsigned long long old = atomicMin(&a.s[ni], nb);
            if (nb < old) {
                const int b = (int)floor(nd);
                if (atomicExch(&a.inq[ni], b + 1) != b + 1) {
                    const unsigned slot = atomicAdd(&a.counts[b % 3], 1u);
                    a.lists[b % 3][slot] = (uint32_t)ni;
                }
            }
        }
    }
}

int fp_field_compute(fp_ctx* ctx, const uint8_t* d_cells) {
    cudaStream_t s = ctx->stream;
    const size_t n = (size_t)ctx->W * (size_t)ctx->H;
    FieldArgs a;
    a.W = ctx->W;
    a.H = ctx->H;
    a.boundary = ctx->boundary;
    a.cells = d_cells;
    a.s = (unsigned long long*)ctx->d_field;
    // Each list holds at most one entry per cell (a cell is queued once per distinct bucket,
    // and a bucket's list is drained before it is reused three buckets later).
    uint32_t* lists = nullptr;
    unsigned int* counts = nullptr;
    int* inq = nullptr;
    FP_CUDA(ctx, cudaMalloc(&lists, 3 * n * sizeof(uint32_t)));
    FP_CUDA(ctx, cudaMalloc(&counts, 4 * sizeof(unsigned int)));
    FP_CUDA(ctx, cudaMalloc(&inq, n * sizeof(int)));
    for (int i = 0; i < 3; ++i) a.lists[i] = lists + (size_t)i * n;
    a.counts = counts;
    a.inq = inq;
    int rc = FP_OK;
    unsigned int* h = nullptr;
    cudaError_t e = cudaMallocHost(&h, 4 * sizeof(unsigned int));
    if (e != cudaSuccess) rc = fp_cuda_fail(ctx, e, "cudaMallocHost");
    if (rc == FP_OK) {
        cudaMemsetAsync(counts, 0, 4 * sizeof(unsigned int), s);
        fp_launch(field_init_kernel, 1184, 256, 0, s, a, n);
        ctx->ctr.kernel_launches++;
        // Process buckets; check for an empty window every `batch` buckets.
        const int batch = 16;
        for (int k = 0;; k += batch) {
            for (int b = k; b < k + batch; ++b) {
                fp_launch(field_relax_kernel, 1184, 256, 0, s, a, b);
                ctx->ctr.kernel_launches++;
                // bucket b is drained; it is reused for b+3
                cudaMemsetAsync(counts + (b % 3), 0, sizeof(unsigned int), s);
            }
            cudaMemcpyAsync(h, counts, 3 * sizeof(unsigned int), cudaMemcpyDeviceToHost, s);
            e = cudaStreamSynchronize(s);
            if (e != cudaSuccess) {
                rc = fp_cuda_fail(ctx, e, "field relaxation");
                break;
            }
            if (h[0] == 0 && h[1] == 0 && h[2] == 0) break;
        }
    }
    if (h) cudaFreeHost(h);
    cudaFree(lists);
    cudaFree(counts);
    cudaFree(inq);
    return rc;
}

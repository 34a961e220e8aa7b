// k_keep.cu -- keep-set bitmasks for the multi-GPU gather: the compressed
// index set of a bin travels as ceil(S/32) 32-bit words (bit s%32 of word s/32, i.e. bit s%8
// of byte s/8 little-endian) instead of S int32 indices, and is expanded back to the
// ascending keep list (Alg. 1 l.16; reading R9) on the receiving side.
#include "dwc_internal.cuh"

namespace dwc {

__global__ void keep_mask_kernel(int S, int words, const int32_t *__restrict__ n_keep,
                                 const int32_t *__restrict__ keep_idx, uint32_t *__restrict__ mask) {
    const int bin = blockIdx.y;
    uint32_t *mb = mask + (size_t)bin * words;
    const int32_t *kb = keep_idx + (size_t)bin * S;
    const int nk = n_keep[bin];
    // word w collects the kept s in [32w, 32w+32): keep list ascending -> binary search the start
    for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < words; w += gridDim.x * blockDim.x) {
        int lo = 0, hi = nk;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (kb[mid] < 32 * w) lo = mid + 1;
            else hi = mid;
        }
        uint32_t bits = 0;
        for (int i = lo; i < nk && kb[i] < 32 * w + 32; i++) bits |= 1u << (kb[i] - 32 * w);
        mb[w] = bits;
    }
}

// one CTA per bin: block-wide exclusive scan of the per-word popcounts, then scatter
constexpr int kUnmaskThreads = 256;
__global__ void __launch_bounds__(kUnmaskThreads)
keep_unmask_kernel(int S, int words, const uint32_t *__restrict__ mask, int32_t *__restrict__ n_keep,
                   int32_t *__restrict__ keep_idx) {
    __shared__ int wsum[kUnmaskThreads / 32];
    __shared__ int carry;
    const int bin = blockIdx.x, tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t *mb = mask + (size_t)bin * words;
    int32_t *kb = keep_idx + (size_t)bin * S;
    if (tid == 0) carry = 0;
    __syncthreads();
    for (int w0 = 0; w0 < words; w0 += kUnmaskThreads) {
        const int w = w0 + tid;
        const uint32_t bits = (w < words) ? mb[w] : 0u;
        const int c = __popc(bits);
        int incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += v;
        }
        if (lane == 31) wsum[wid] = incl;
        __syncthreads();
        int before = carry;
        for (int q = 0; q < wid; q++) before += wsum[q];
        int pos = before + incl - c;
        for (uint32_t b = bits; b; b &= b - 1) kb[pos++] = 32 * w + __ffs(b) - 1;
        __syncthreads();
        if (tid == kUnmaskThreads - 1) carry = before + incl;
        __syncthreads();
    }
    const int total = carry;
    for (int i = total + tid; i < S; i += kUnmaskThreads) kb[i] = -1;
    if (tid == 0) n_keep[bin] = total;
}

int launch_keep_mask(int n_bins, int S, const int32_t *n_keep, const int32_t *keep_idx, uint32_t *mask,
                     cudaStream_t st) {
    const int words = (S + 31) / 32;
    dim3 grid((words + 127) / 128, n_bins);
    keep_mask_kernel<<<grid, 128, 0, st>>>(S, words, n_keep, keep_idx, mask);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

int launch_keep_unmask(int n_bins, int S, const uint32_t *mask, int32_t *n_keep, int32_t *keep_idx,
                       cudaStream_t st) {
    keep_unmask_kernel<<<n_bins, kUnmaskThreads, 0, st>>>(S, (S + 31) / 32, mask, n_keep, keep_idx);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

// dwc_gs precondition: every A_ii > 0 and finite; sets bit 2 of *flag otherwise.
// Bit 4: some entry has its sign bit set or is not finite (the residual kernel then widens A~
// with F2F instead of its non-negative bit placement).
__global__ void diag_check_kernel(int n, const float *__restrict__ A, int *__restrict__ flag) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const float v = A[(size_t)i * n + i];
        if (!(v > 0.f) || !isfinite(v)) atomicOr(flag, 2);
    }
    bool neg = false;
    const size_t nn = (size_t)n * n;
    for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < nn; e += (size_t)gridDim.x * blockDim.x) {
        const float v = A[e];
        neg |= (__float_as_uint(v) >> 31) != 0u || !isfinite(v);
    }
    if (__any_sync(0xffffffffu, neg) && (threadIdx.x & 31) == 0) atomicOr(flag, 4);
}

int launch_diag_check(int n, const float *A, int *flag, cudaStream_t st) {
    diag_check_kernel<<<148, 256, 0, st>>>(n, A, flag);
    return cudaPeekAtLastError() == cudaSuccess ? 1 : -1;
}

}  // namespace dwc

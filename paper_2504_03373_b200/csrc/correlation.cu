// Kernel (1): sliding-window spatial correlation R(w) = (1/T) sum X X^H.
//
// Follows CorrelationWindow (reference proj/src/correlation.cpp:53-130):
// an FP64 running sum over the full M x M matrix, updated per push by
// subtracting the frame leaving the window and adding the new one
// (correlation.cpp:103-106), rebuilt oldest-first every `rebuild_interval`
// pushes (75-84), and normalized as float(sum * (1/T)) (112-130).
//
// Bit-exactness: X entries are float, so every product of two entries is
// exact in double; the only roundings are (a*c + b*d), the running-sum add and
// the final scale/narrow.  They are issued with explicit _rn intrinsics so the
// compiler cannot contract them differently, which makes R bit-identical to
// the reference's for the same push sequence.
//
// Layout: one CTA per frequency bin; each thread owns up to kPer entries of
// that bin's M x M running sum in registers for the whole launch, so the FP64
// state is read and written once per launch however many frames it ingests.
// The frames of a launch are consumed in order (the recurrence is sequential
// in time); parallelism is over bins x matrix entries.
#include "common.cuh"
#include "kernels.cuh"

namespace sslg {

constexpr int kCorrThreads = 512;
constexpr int kCorrPer = (kMaxM * kMaxM + kCorrThreads - 1) / kCorrThreads;  // 8
constexpr int kCorrChunk = 32;  // frames staged per pass

__device__ __forceinline__ void outer_acc(double2& acc, float2 xi, float2 xj, bool subtract) {
    const double a = xi.x, b = xi.y, c = xj.x, d = xj.y;
    // xi * conj(xj): (a*c + b*d, b*c - a*d), one rounding each (products exact)
    const double re = __fma_rn(a, c, __dmul_rn(b, d));
    const double im = __fma_rn(b, c, -__dmul_rn(a, d));
    if (subtract) {
        acc.x = __dadd_rn(acc.x, -re);
        acc.y = __dadd_rn(acc.y, -im);
    } else {
        acc.x = __dadd_rn(acc.x, re);
        acc.y = __dadd_rn(acc.y, im);
    }
}

// NT threads own up to PER entries each: 512 x 8 for the full m <= 64, and
// for small arrays just enough warps to cover the m x m entries once (C1:
// 64 threads; the 512-thread form spent 87% of its issue slots on warps
// that own no entry).
template <int NT, int PER>
__global__ void __launch_bounds__(NT, NT >= 512 ? 2 : 1) correlation_kernel(CorrArgs a) {
    if (a.abort && *a.abort) return;  // skipped after a failed asynchronous gate
    __shared__ float2 xs_new[kMaxM];
    __shared__ float2 xc_new[kCorrChunk * kMaxM];
    __shared__ float2 xc_old[kCorrChunk * kMaxM];
    const int b = blockIdx.x;
    const int m = a.m;
    const int mm = m * m;
    const int tid = threadIdx.x;

    double2 acc[PER];
    int eij[PER];  // (row << 8) | column of each owned entry
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const int e = tid + k * NT;
        eij[k] = ((e / m) << 8) | (e % m);
        acc[k] = e < mm ? a.state[(size_t)b * mm + e] : make_double2(0, 0);
    }
    const double inv_t = 1.0 / (double)a.t;
    long long pushed = a.pushed0;
    long long since = a.since0;
    long long first_emit = (long long)a.t - 1 - a.pushed0;
    if (first_emit < 0) first_emit = 0;

    auto frame_ptr = [&](long long g) { return a.ring + (size_t)(g % a.cap) * m * a.bins; };

    // the bin's entering and leaving frame values for up to kCorrChunk frames
    // are staged together up front, so the sequential recurrence below never
    // waits on a global load
    for (int f0 = 0; f0 < a.frames; f0 += kCorrChunk) {
        const int nf = min(kCorrChunk, a.frames - f0);
        __syncthreads();
        for (int x = tid; x < nf * m; x += NT) {
            const int fi = x / m, ch = x - fi * m;
            const long long g = a.pushed0 + f0 + fi;
            xc_new[x] = frame_ptr(g)[(size_t)ch * a.bins + b];
            if (g >= a.t) xc_old[x] = frame_ptr(g - a.t)[(size_t)ch * a.bins + b];
        }
        __syncthreads();
        for (int fi = 0; fi < nf; ++fi) {
            const int f = f0 + fi;
            const bool drop_old = pushed >= a.t;
            const float2* xn = xc_new + fi * m;
            const float2* xo = xc_old + fi * m;
#pragma unroll
            for (int k = 0; k < PER; ++k) {
                if (tid + k * NT < mm) {
                    if (drop_old) outer_acc(acc[k], xo[eij[k] >> 8], xo[eij[k] & 255], true);
                    outer_acc(acc[k], xn[eij[k] >> 8], xn[eij[k] & 255], false);
                }
            }
            ++pushed;
            if (++since >= a.rebuild_interval) {
                // rebuild oldest first (correlation.cpp:75-84)
                const long long have = pushed < a.t ? pushed : a.t;
#pragma unroll
                for (int k = 0; k < PER; ++k) acc[k] = make_double2(0, 0);
                for (long long kk = 0; kk < have; ++kk) {
                    const long long gg = pushed - have + kk;
                    __syncthreads();
                    if (tid < m) xs_new[tid] = frame_ptr(gg)[(size_t)tid * a.bins + b];
                    __syncthreads();
#pragma unroll
                    for (int k = 0; k < PER; ++k)
                        if (tid + k * NT < mm) outer_acc(acc[k], xs_new[eij[k] >> 8], xs_new[eij[k] & 255], false);
                }
                since = 0;
            }
            if (f >= first_emit) {
                float2* r = a.r_out + ((size_t)(f - first_emit) * a.bins + b) * mm;
#pragma unroll
                for (int k = 0; k < PER; ++k) {
                    const int e = tid + k * NT;
                    if (e < mm)
                        r[e] = make_float2(__double2float_rn(__dmul_rn(acc[k].x, inv_t)),
                                           __double2float_rn(__dmul_rn(acc[k].y, inv_t)));
                }
            }
        }
    }
#pragma unroll
    for (int k = 0; k < PER; ++k) {
        const int e = tid + k * NT;
        if (e < mm) a.state[(size_t)b * mm + e] = acc[k];
    }
}

// Non-finite guard (correlation.cpp:90-95): counts non-finite spectrum values
// of the frames about to be ingested.
__global__ void count_nonfinite_kernel(const float* p, size_t n, unsigned int* bad) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    unsigned int local = 0;
    for (; i < n; i += stride) local += isfinite(p[i]) ? 0u : 1u;
    if (local) atomicAdd(bad, local);
}

__global__ void gate_abort_kernel(const float* p, size_t n, unsigned int* abort, unsigned int id) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    bool bad = false;
    for (; i < n; i += stride) bad |= !isfinite(p[i]);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicCAS(abort, 0u, id + 1u);
}

void launch_gate_abort(const float* p, size_t n, unsigned int* abort, unsigned int id, cudaStream_t s) {
    const int threads = 256;
    size_t blocks = (n + threads - 1) / threads;
    if (blocks > 1024) blocks = 1024;
    if (blocks == 0) blocks = 1;
    gate_abort_kernel<<<(unsigned)blocks, threads, 0, s>>>(p, n, abort, id);
}

void launch_correlation(const CorrArgs& a, cudaStream_t s) {
    const int mm = a.m * a.m;
    if (mm <= 64) {
        correlation_kernel<64, 1><<<a.bins, 64, 0, s>>>(a);
    } else if (mm <= 256) {
        correlation_kernel<256, 1><<<a.bins, 256, 0, s>>>(a);
    } else {
        correlation_kernel<kCorrThreads, kCorrPer><<<a.bins, kCorrThreads, 0, s>>>(a);
    }
}

void launch_count_nonfinite(const float* p, size_t n, unsigned int* bad, cudaStream_t s) {
    const int threads = 256;
    size_t blocks = (n + threads - 1) / threads;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks == 0) blocks = 1;
    count_nonfinite_kernel<<<(unsigned)blocks, threads, 0, s>>>(p, n, bad);
}

// Per-frame gate of the synchronous paths: the smallest index (frame0 + f)
// of a frame holding a non-finite value lands in *first (atomicMin; the
// caller initializes it to 0xffffffff).  CorrelationWindow::push rejects
// exactly that frame (correlation.cpp:16-17) and keeps every earlier one.
__global__ void first_nonfinite_kernel(const float* p, size_t per_frame, int nframes, unsigned int frame0,
                                       unsigned int* first) {
    const size_t n = per_frame * (size_t)nframes;
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    unsigned int best = 0xffffffffu;
    for (; i < n; i += stride)
        if (!isfinite(p[i])) {
            const unsigned int f = frame0 + (unsigned int)(i / per_frame);
            best = f < best ? f : best;
        }
    for (int o = 16; o; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
    if ((threadIdx.x & 31) == 0 && best != 0xffffffffu) atomicMin(first, best);
}

void launch_first_nonfinite(const float* p, size_t per_frame, int nframes, unsigned int frame0, unsigned int* first,
                            cudaStream_t s) {
    const int threads = 256;
    size_t blocks = (per_frame * (size_t)nframes + threads - 1) / threads;
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks == 0) blocks = 1;
    first_nonfinite_kernel<<<(unsigned)blocks, threads, 0, s>>>(p, per_frame, nframes, frame0, first);
}

}  // namespace sslg

// Kernels (3) and (4): MUSIC pseudo-spectrum, broadband integration, peaks.
//
// (3) P(theta, w) = |h|^2 / max(floor, sum_{i >= Ns} |h^H e_i|)
//     (calc_average_power, reference proj/src/music.cpp:112-165; squared
//     denominator optional, music.hpp:55-57), FP64 arithmetic on the FP32
//     steering table.  One CTA per (block, bin, direction chunk): the bin's
//     noise vectors E_n (FP64) and the chunk's steering vectors (transposed to
//     [mic][dir] so consecutive threads read consecutive directions) are staged
//     in SMEM; thread (direction, part) accumulates |h^H e_i| over its share of
//     the noise vectors four at a time (one steering load feeds four complex
//     FMAs).  Every direction runs the identical instruction sequence, so
//     bit-identical steering vectors give bit-identical powers (exact ties
//     survive to the peak search, music.cpp:215-223).
// (4) Pbar(theta) = sum_w P(theta, w) in ascending-bin FP64 order
//     (music.cpp:160), then the local-maximum test on the host-built neighbor
//     topology, stable (power desc, index asc) top-Ns and the low-power flag
//     against the sequential FP64 mean (peak_search, music.cpp:197-236).
#include "common.cuh"
#include "kernels.cuh"

namespace sslg {

constexpr int kSpecThreads = 256;
constexpr int kSpecVec = 4;  // noise vectors per steering load

__global__ void __launch_bounds__(kSpecThreads) spectrum_kernel(SpecArgs a) {
    if (a.abort && *a.abort) return;  // skipped after a failed asynchronous gate
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int m = a.m;
    const int nn = m - a.ns;
    double2* En = reinterpret_cast<double2*>(smem_raw);             // [nn][m]
    float2* Hs = reinterpret_cast<float2*>(En + (size_t)nn * m);   // [m][dchunk]
    double* part_den = reinterpret_cast<double*>(Hs + (size_t)m * a.dchunk);  // [nsplit][dchunk]

    const int blkbin = blockIdx.x;  // block * bins + bin
    const int bin = blkbin % a.bins;
    const int d0 = blockIdx.y * a.dchunk;
    const int nd = min(a.dchunk, a.dirs - d0);
    const int t = threadIdx.x;

    const double2* eb = a.e + ((size_t)blkbin * m + a.ns) * m;
    for (int x = t; x < nn * m; x += blockDim.x) En[x] = eb[x];
    const float2* hb = a.h + ((size_t)bin * a.dirs + d0) * m;
    for (int x = t; x < nd * m; x += blockDim.x) {
        const int d = x / m, mic = x % m;
        Hs[mic * a.dchunk + d] = hb[x];
    }
    __syncthreads();

    const int d = t % a.dchunk;
    const int part = t / a.dchunk;
    if (part < a.nsplit && d < nd) {
        double den = 0;
        // vector chunks of kSpecVec assigned round-robin to parts
        for (int v0 = part * kSpecVec; v0 < nn; v0 += a.nsplit * kSpecVec) {
            double2 acc[kSpecVec];
#pragma unroll
            for (int u = 0; u < kSpecVec; ++u) acc[u] = make_double2(0, 0);
            for (int mic = 0; mic < m; ++mic) {
                const double2 hv = f2d(Hs[mic * a.dchunk + d]);
#pragma unroll
                for (int u = 0; u < kSpecVec; ++u)
                    if (v0 + u < nn) acc[u] = cadd(acc[u], cmulc(hv, En[(v0 + u) * m + mic]));
            }
#pragma unroll
            for (int u = 0; u < kSpecVec; ++u) {
                if (v0 + u < nn) {
                    const double mag = hypot(acc[u].x, acc[u].y);
                    den += a.squared ? mag * mag : mag;
                }
            }
        }
        part_den[part * a.dchunk + d] = den;
    }
    __syncthreads();
    if (t < nd) {
        double den = part_den[t];
        for (int pp = 1; pp < a.nsplit; ++pp) den += part_den[pp * a.dchunk + t];
        if (den < a.floor_) den = a.floor_;
        const double num = a.num[(size_t)bin * a.dirs + d0 + t];
        a.p[(size_t)blkbin * a.dirs + d0 + t] = num / den;
    }
}


// Register-tiled variant for large grids (C4: 1368 directions): each thread
// owns a 4-direction x 4-vector tile of h^H e products, so one mic step loads
// 4 steering + 4 noise values for 16 complex MACs (64 FP64 FMAs).  The noise
// vectors are staged transposed ([mic][vector], padded to 64) and the
// steering chunk as [mic][direction], so a warp's loads are contiguous and
// conflict-free.  The 16 threads holding the same directions and different
// vector slices are adjacent lanes; their partial denominators meet in a
// 4-level shuffle tree, identical for every direction (exact ties survive).
constexpr int kTileD = 4, kTileN = 4, kSlices = 16;
constexpr int kNPad = kTileN * kSlices;      // 64 vector slots
constexpr int kEStride = kNPad + 1;          // double2 row stride of the staged noise vectors (bank spread)

// DT direction tiles of 4 per CTA (16 lanes each): 64 directions at DT = 16
// (large grids), the whole 72-direction ring at DT = 18.
template <int DT>
__global__ void __launch_bounds__(16 * DT, 2) spectrum_tiled_kernel(SpecArgs a, int nblk, int nchunk) {
    constexpr int kChunk2 = kTileD * DT;
    constexpr int kHStride = kChunk2 + 2;  // float2 row stride of the staged steering (16-B aligned rows)
    if (a.abort && *a.abort) return;  // skipped after a failed asynchronous gate
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int m = a.m;
    const int nn = m - a.ns;
    double2* Et = reinterpret_cast<double2*>(smem_raw);                 // [m][kEStride]
    float2* Hs = reinterpret_cast<float2*>(Et + (size_t)m * kEStride);  // [m][kHStride]
    // linear CTA index = (bin * nblk + block) * nchunk + chunk: the chunks of
    // one (block, bin) run back to back (its noise vectors stay in L2) and
    // the blocks of one bin follow each other (its steering stays in L2)
    const int chunk = blockIdx.x % nchunk;
    const int bb = blockIdx.x / nchunk;
    const int bin = bb / nblk, blk = bb % nblk;
    const int blkbin = blk * a.bins + bin;
    const int d0 = chunk * kChunk2;
    const int nd = min(kChunk2, a.dirs - d0);
    const int t = threadIdx.x;

    // staging: coalesced global reads, transposed shared writes (padded strides)
    const double2* eb = a.e + ((size_t)blkbin * m + a.ns) * m;  // [nn][m]
    for (int x = t; x < kNPad * m; x += blockDim.x) {
        const int v = x / m, mic = x % m;
        Et[mic * kEStride + v] = v < nn ? eb[(size_t)v * m + mic] : make_double2(0, 0);
    }
    const float2* hb = a.h + ((size_t)bin * a.dirs + d0) * m;
    for (int x = t; x < kChunk2 * m; x += blockDim.x) {
        const int d = x / m, mic = x % m;
        Hs[mic * kHStride + d] = d < nd ? hb[(size_t)d * m + mic] : make_float2(0.f, 0.f);
    }
    __syncthreads();

    const int slice = t % kSlices, dtile = t / kSlices;
    double2 acc[kTileD][kTileN];
#pragma unroll
    for (int i = 0; i < kTileD; ++i)
#pragma unroll
        for (int j = 0; j < kTileN; ++j) acc[i][j] = make_double2(0, 0);
    const float2* hrow = Hs + dtile * kTileD;
    const double2* erow = Et + slice;  // vectors slice, slice + 16, ...: lanes read consecutive 16 B
#pragma unroll 2
    for (int mic = 0; mic < m; ++mic) {
        const float4 h01 = *reinterpret_cast<const float4*>(hrow + mic * kHStride);
        const float4 h23 = *reinterpret_cast<const float4*>(hrow + mic * kHStride + 2);
        const double2 h[kTileD] = {make_double2(h01.x, h01.y), make_double2(h01.z, h01.w),
                                   make_double2(h23.x, h23.y), make_double2(h23.z, h23.w)};
        double2 e[kTileN];
#pragma unroll
        for (int j = 0; j < kTileN; ++j) e[j] = erow[mic * kEStride + j * kSlices];
#pragma unroll
        for (int i = 0; i < kTileD; ++i)
#pragma unroll
            for (int j = 0; j < kTileN; ++j) {  // conj(h) e
                acc[i][j].x = fma(h[i].x, e[j].x, fma(h[i].y, e[j].y, acc[i][j].x));
                acc[i][j].y = fma(h[i].x, e[j].y, fma(-h[i].y, e[j].x, acc[i][j].y));
            }
    }
    double den[kTileD];
#pragma unroll
    for (int i = 0; i < kTileD; ++i) {
        double sum = 0;
#pragma unroll
        for (int j = 0; j < kTileN; ++j) {
            const double mag = hypot(acc[i][j].x, acc[i][j].y);
            sum += a.squared ? mag * mag : mag;
        }
        den[i] = sum;
    }
#pragma unroll
    for (int o = kSlices / 2; o > 0; o >>= 1)
#pragma unroll
        for (int i = 0; i < kTileD; ++i) den[i] += __shfl_xor_sync(0xffffffffu, den[i], o);
    if (slice < kTileD) {
        const int d = dtile * kTileD + slice;
        double dd = den[0];
#pragma unroll
        for (int i = 1; i < kTileD; ++i)
            if (slice == i) dd = den[i];
        if (d < nd) {
            if (dd < a.floor_) dd = a.floor_;
            const double num = a.num[(size_t)bin * a.dirs + d0 + d];
            a.p[(size_t)blkbin * a.dirs + d0 + d] = num / dd;
        }
    }
}

// |h|^2 per (bin, dir) in the reference's order: sequential over mics,
// (re^2 + im^2) rounded once (both squares exact in double).
__global__ void steering_prep_kernel(const float2* __restrict__ h_in,  // [dirs][bins][m]
                                     float2* __restrict__ h_t,         // [bins][dirs][m]
                                     double* __restrict__ num, int m, int bins, int dirs) {
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)bins * dirs) return;
    const int b = (int)(idx / dirs), d = (int)(idx % dirs);
    const float2* src = h_in + ((size_t)d * bins + b) * m;
    float2* dst = h_t + ((size_t)b * dirs + d) * m;
    double acc = 0;
    for (int mic = 0; mic < m; ++mic) {
        const float2 v = src[mic];
        dst[mic] = v;
        const double re = v.x, im = v.y;
        acc = __dadd_rn(acc, __fma_rn(re, re, __dmul_rn(im, im)));
    }
    num[idx] = acc;
}

constexpr int kPeakThreads = 256;

__global__ void __launch_bounds__(kPeakThreads) integrate_peaks_kernel(PeakArgs a) {
    if (a.abort && *a.abort) return;  // skipped after a failed asynchronous gate
    extern __shared__ __align__(16) unsigned char smem_raw[];
    double* pw = reinterpret_cast<double*>(smem_raw);              // [dirs]
    int* is_peak = reinterpret_cast<int*>(pw + a.dirs);            // [dirs]
    __shared__ double s_mean;
    const int blk = blockIdx.x;
    const int t = threadIdx.x;
    const double* pb = a.p + (size_t)blk * a.bins * a.dirs;
    for (int d = t; d < a.dirs; d += blockDim.x) {
        double acc = 0.0;
        for (int b = 0; b < a.bins; ++b) acc = __dadd_rn(acc, pb[(size_t)b * a.dirs + d]);
        pw[d] = acc;
        a.power[(size_t)blk * a.dirs + d] = acc;
    }
    __syncthreads();
    if (t == 0) {
        double mean = 0;
        for (int d = 0; d < a.dirs; ++d) mean = __dadd_rn(mean, pw[d]);
        if (a.dirs) mean = __ddiv_rn(mean, (double)a.dirs);
        s_mean = mean;
    }
    for (int d = t; d < a.dirs; d += blockDim.x) {
        int ok = 1;
        for (uint32_t k = a.nbr_off[d]; k < a.nbr_off[d + 1]; ++k)
            if (pw[d] < pw[a.nbr[k]]) {
                ok = 0;
                break;
            }
        is_peak[d] = ok;
    }
    __syncthreads();
    if (t == 0) {
        // insertion into a bounded list ordered by (power desc, index asc);
        // peaks are visited in index order, so equal powers keep index order
        uint32_t best[64];
        int nb = 0;
        const int cap = a.ns < 64 ? a.ns : 64;
        for (int d = 0; d < a.dirs; ++d) {
            if (!is_peak[d]) continue;
            const double v = pw[d];
            int pos = nb;
            while (pos > 0 && v > pw[best[pos - 1]]) --pos;
            if (pos >= cap) continue;
            const int last = nb < cap ? nb : cap - 1;
            for (int k = last; k > pos; --k) best[k] = best[k - 1];
            best[pos] = (uint32_t)d;
            if (nb < cap) ++nb;
        }
        const double thr = a.low_ratio * s_mean;
        for (int k = 0; k < nb; ++k) {
            a.est_idx[(size_t)blk * a.ns + k] = best[k];
            a.est_pw[(size_t)blk * a.ns + k] = pw[best[k]];
            a.est_low[(size_t)blk * a.ns + k] = pw[best[k]] < thr ? 1 : 0;
        }
        for (int k = nb; k < a.ns; ++k) {  // unused slots: no estimate
            a.est_idx[(size_t)blk * a.ns + k] = 0xffffffffu;
            a.est_pw[(size_t)blk * a.ns + k] = 0.0;
            a.est_low[(size_t)blk * a.ns + k] = 0;
        }
        a.est_count[blk] = (uint32_t)nb;
    }
}

void spectrum_shape(int m, int ns, int dirs, int& dchunk, int& nsplit, size_t& smem) {
    dchunk = dirs < 128 ? dirs : 128;
    nsplit = kSpecThreads / dchunk;
    const int nn = m - ns;
    const int max_split = (nn + kSpecVec - 1) / kSpecVec;
    if (nsplit > max_split) nsplit = max_split;
    if (nsplit < 1) nsplit = 1;
    smem = (size_t)nn * m * sizeof(double2) + (size_t)m * dchunk * sizeof(float2) +
           (size_t)nsplit * dchunk * sizeof(double);
}

void launch_spectrum(SpecArgs a, int nblk, cudaStream_t s) {
    auto tiled = [&](auto kern, int dt) {
        const int chunk = kTileD * dt;
        const size_t smem2 = (size_t)a.m * kEStride * sizeof(double2) + (size_t)a.m * (chunk + 2) * sizeof(float2);
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
        const int nchunk = (a.dirs + chunk - 1) / chunk;
        kern<<<nblk * a.bins * nchunk, 16 * dt, smem2, s>>>(a, nblk, nchunk);
    };
    // register-tiled kernel: 16 slices of 4 noise vectors per direction, so
    // it needs enough noise vectors to fill them (C1/C2, with 6 and 14, run
    // 3.5x faster on the generic kernel)
    if (a.m - a.ns <= kNPad && a.m - a.ns >= 32) {
        if (a.dirs >= 256) {
            tiled(spectrum_tiled_kernel<16>, 16);
            return;
        }
        if (a.dirs > 64 && a.dirs <= 72) {
            tiled(spectrum_tiled_kernel<18>, 18);
            return;
        }
    }
    size_t smem;
    spectrum_shape(a.m, a.ns, a.dirs, a.dchunk, a.nsplit, smem);
    cudaFuncSetAttribute(spectrum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    dim3 grid(nblk * a.bins, (a.dirs + a.dchunk - 1) / a.dchunk);
    spectrum_kernel<<<grid, kSpecThreads, smem, s>>>(a);
}

void launch_steering_prep(const float2* h_in, float2* h_t, double* num, int m, int bins, int dirs,
                          cudaStream_t s) {
    const size_t n = (size_t)bins * dirs;
    steering_prep_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(h_in, h_t, num, m, bins, dirs);
}

void launch_peaks(const PeakArgs& a, int nblk, cudaStream_t s) {
    const size_t smem = (size_t)a.dirs * (sizeof(double) + sizeof(int));
    cudaFuncSetAttribute(integrate_peaks_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    integrate_peaks_kernel<<<nblk, kPeakThreads, smem, s>>>(a);
}

}  // namespace sslg

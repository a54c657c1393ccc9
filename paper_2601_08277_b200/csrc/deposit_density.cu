// deposit_density.cu -- bit-exact charge density (pic::deposit_density,
// proj/include/pic/deposit.hpp:76-83).
//
// The reference scatters quantity[p]*S in STORAGE order, so node n's value is
// the left-to-right sum of its contributions ordered by storage index.  A GPU
// scatter (atomics or per-cell partials) reorders that sum (SURVEY Appendix
// A.3: 507/756 and 650/756 nodes differ).  This file is an ordered GATHER: a
// thread owns one node and visits exactly the particles that touch it, in
// storage order, with round-to-nearest intrinsics (no FMA contraction):
//
//  * sorted storage (the session's bins, or any cell-sorted store): the
//    contributions of node n come from its W^3 source cells; storage order is
//    then "source cells by ascending linear id, then slot order".  Per axis
//    the W wrapped source indices are sorted once; nested k->j->i loops over
//    the sorted lists visit cells in ascending linear id (grid.hpp:50-54).
//  * unsorted storage (stateless calls on arbitrary arrays): a k-way merge of
//    the W^3 per-cell lists by storage rank.
//
// Value order per contribution: wq * (sx[ix] * (sy[jy] * sz[kz])), exactly
// scatter_deposit's (deposit.hpp:41-48).
#include "common.cuh"
#include "kernels.hpp"

namespace picgpu {

namespace {

template <int ORDER>
__global__ void density_prologue(const GridD g, const CSoa p, const double* __restrict__ quantity, double qscale,
                                 uint64_t slots, double* __restrict__ S, uint8_t* __restrict__ upb) {
    constexpr int W = Shape<ORDER>::W;
    const uint64_t s = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= slots) return;
    const double x = p.x[s], y = p.y[s], z = p.z[s];
    double f[3];
    locate_x(g, x, f[0]);
    locate_axis(y, g.oy, g.dy, g.inv_dy, g.pow2y, g.ny, f[1]);
    locate_axis(z, g.oz, g.dz, g.inv_dz, g.pow2z, g.nz, f[2]);
    int bits = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        double w[W];
        int up;
        Shape<ORDER>::weights(f[a], w, up);
        bits |= up << a;
#pragma unroll
        for (int t = 0; t < W; ++t) S[(size_t)(a * W + t) * slots + s] = w[t];
    }
    S[(size_t)(3 * W) * slots + s] = quantity ? quantity[s] : qscale * p.w[s];
    if (ORDER == 2) upb[s] = (uint8_t)bits;
}

// Sorted list of the W wrapped source indices of node coordinate X along one
// axis: src = wrap(X - OFF - t), tap t (node = cell + OFF + t).
template <int W, int OFF>
__device__ __forceinline__ void sources(int X, int n, int (&src)[W], int (&tap)[W]) {
#pragma unroll
    for (int t = 0; t < W; ++t) {
        src[t] = wrap_index(X - OFF - t, n);
        tap[t] = t;
    }
    // tiny insertion sort (W <= 4), ascending by src
#pragma unroll
    for (int a = 1; a < W; ++a)
#pragma unroll
        for (int b = a; b > 0; --b)
            if (src[b] < src[b - 1]) {
                const int ts = src[b]; src[b] = src[b - 1]; src[b - 1] = ts;
                const int tt = tap[b]; tap[b] = tap[b - 1]; tap[b - 1] = tt;
            }
}

// TSC pads 3 taps into the 4-wide window; the padded tap must be skipped, not
// added as zero (keeps -0.0 / +0.0 identical to the 27-tap reference loop).
template <int ORDER>
__device__ __forceinline__ bool tap_valid(int up, int t) {
    if (ORDER != 2) return true;
    return up ? t != 0 : t != 3;
}

template <int ORDER>
__global__ void density_gather_sorted(const GridD g, const uint32_t* __restrict__ off,
                                      const uint32_t* __restrict__ cnt, const double* __restrict__ S, uint64_t slots,
                                      const uint8_t* __restrict__ upb, double* __restrict__ rho) {
    constexpr int W = Shape<ORDER>::W, OFF = Shape<ORDER>::OFF;
    const uint64_t node = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (node >= g.ncells) return;
    const int X = (int)(node % (uint32_t)g.nx);
    const int Y = (int)((node / (uint32_t)g.nx) % (uint32_t)g.ny);
    const int Z = (int)(node / ((uint64_t)g.nx * (uint32_t)g.ny));
    int xs[W], xt[W], ys[W], yt[W], zs[W], zt[W];
    sources<W, OFF>(X, g.nx, xs, xt);
    sources<W, OFF>(Y, g.ny, ys, yt);
    sources<W, OFF>(Z, g.nz, zs, zt);
    const double* SQ = S + (size_t)(3 * W) * slots;
    double acc = 0.0;
    for (int zi = 0; zi < W; ++zi) {
        const double* Sz = S + (size_t)(2 * W + zt[zi]) * slots;
        for (int yi = 0; yi < W; ++yi) {
            const double* Sy = S + (size_t)(W + yt[yi]) * slots;
            const uint32_t row = (uint32_t)g.nx * ((uint32_t)ys[yi] + (uint32_t)g.ny * (uint32_t)zs[zi]);
            for (int xi = 0; xi < W; ++xi) {
                const double* Sx = S + (size_t)xt[xi] * slots;
                const uint32_t c = (uint32_t)xs[xi] + row;
                const uint32_t o = off[c], n = cnt[c];
                for (uint32_t u = 0; u < n; ++u) {
                    const uint32_t s = o + u;
                    if (ORDER == 2) {
                        const int b = upb[s];
                        if (!tap_valid<ORDER>(b & 1, xt[xi]) || !tap_valid<ORDER>((b >> 1) & 1, yt[yi]) ||
                            !tap_valid<ORDER>((b >> 2) & 1, zt[zi]))
                            continue;
                    }
                    const double syz = __dmul_rn(Sy[s], Sz[s]);
                    const double sv = __dmul_rn(Sx[s], syz);
                    acc = __dadd_rn(acc, __dmul_rn(SQ[s], sv));
                }
            }
        }
    }
    rho[node] = acc;
}

template <int ORDER>
__global__ void density_gather_merge(const GridD g, const uint32_t* __restrict__ off, const uint32_t* __restrict__ cnt,
                                     const uint32_t* __restrict__ rank, const double* __restrict__ S, uint64_t slots,
                                     const uint8_t* __restrict__ upb, double* __restrict__ rho) {
    constexpr int W = Shape<ORDER>::W, OFF = Shape<ORDER>::OFF;
    constexpr int NC = W * W * W;
    const uint64_t node = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (node >= g.ncells) return;
    const int X = (int)(node % (uint32_t)g.nx);
    const int Y = (int)((node / (uint32_t)g.nx) % (uint32_t)g.ny);
    const int Z = (int)(node / ((uint64_t)g.nx * (uint32_t)g.ny));
    int xs[W], xt[W], ys[W], yt[W], zs[W], zt[W];
    sources<W, OFF>(X, g.nx, xs, xt);
    sources<W, OFF>(Y, g.ny, ys, yt);
    sources<W, OFF>(Z, g.nz, zs, zt);
    uint32_t head[NC], end[NC];
    int taps[NC];
#pragma unroll
    for (int zi = 0; zi < W; ++zi)
#pragma unroll
        for (int yi = 0; yi < W; ++yi)
#pragma unroll
            for (int xi = 0; xi < W; ++xi) {
                const int l = (zi * W + yi) * W + xi;
                const uint32_t c =
                    (uint32_t)xs[xi] + (uint32_t)g.nx * ((uint32_t)ys[yi] + (uint32_t)g.ny * (uint32_t)zs[zi]);
                head[l] = off[c];
                end[l] = off[c] + cnt[c];
                taps[l] = xt[xi] | (yt[yi] << 4) | (zt[zi] << 8);
            }
    const double* SQ = S + (size_t)(3 * W) * slots;
    double acc = 0.0;
    for (;;) {
        int best = -1;
        uint32_t br = 0xffffffffu;
        for (int l = 0; l < NC; ++l)
            if (head[l] < end[l]) {
                const uint32_t r = rank[head[l]];
                if (r < br) {
                    br = r;
                    best = l;
                }
            }
        if (best < 0) break;
        const uint32_t s = head[best]++;
        const int tx = taps[best] & 15, ty = (taps[best] >> 4) & 15, tz = taps[best] >> 8;
        if (ORDER == 2) {
            const int b = upb[s];
            if (!tap_valid<ORDER>(b & 1, tx) || !tap_valid<ORDER>((b >> 1) & 1, ty) ||
                !tap_valid<ORDER>((b >> 2) & 1, tz))
                continue;
        }
        const double syz = __dmul_rn(S[(size_t)(W + ty) * slots + s], S[(size_t)(2 * W + tz) * slots + s]);
        const double sv = __dmul_rn(S[(size_t)tx * slots + s], syz);
        acc = __dadd_rn(acc, __dmul_rn(SQ[s], sv));
    }
    rho[node] = acc;
}

template <int ORDER>
void prologue(const GridD& g, const CSoa& p, const double* quantity, double qscale, uint64_t slots, void* scratch,
              cudaStream_t st, double*& S, uint8_t*& upb) {
    constexpr int W = Shape<ORDER>::W;
    S = static_cast<double*>(scratch);
    upb = reinterpret_cast<uint8_t*>(S + (size_t)(3 * W + 1) * slots);
    if (slots == 0) return;
    density_prologue<ORDER><<<div_up((long long)slots, 256), 256, 0, st>>>(g, p, quantity, qscale, slots, S, upb);
    note_launch();
    PICGPU_CUDA_TRY(cudaGetLastError());
}

template <int ORDER>
void run_sorted(const GridD& g, const CSoa& p, const double* quantity, double qscale, const uint32_t* off, const uint32_t* cnt,
                uint64_t slots, void* scratch, double* rho, cudaStream_t st) {
    double* S;
    uint8_t* upb;
    prologue<ORDER>(g, p, quantity, qscale, slots, scratch, st, S, upb);
    density_gather_sorted<ORDER><<<div_up(g.ncells, 128), 128, 0, st>>>(g, off, cnt, S, slots, upb, rho);
    note_launch();
    PICGPU_CUDA_TRY(cudaGetLastError());
}

template <int ORDER>
void run_merge(const GridD& g, const CSoa& p, const double* quantity, double qscale, const uint32_t* rank, const uint32_t* off,
               const uint32_t* cnt, uint64_t slots, void* scratch, double* rho, cudaStream_t st) {
    double* S;
    uint8_t* upb;
    prologue<ORDER>(g, p, quantity, qscale, slots, scratch, st, S, upb);
    density_gather_merge<ORDER><<<div_up(g.ncells, 128), 128, 0, st>>>(g, off, cnt, rank, S, slots, upb, rho);
    note_launch();
    PICGPU_CUDA_TRY(cudaGetLastError());
}

}  // namespace

size_t density_scratch_bytes(int order, uint64_t slots) {
    const int W = order == 1 ? 2 : 4;
    return (size_t)(3 * W + 1) * slots * sizeof(double) + slots + 16;
}

void launch_deposit_density(int order, const GridD& g, const CSoa& p, const double* quantity, double qscale,
                            const uint32_t* off,
                            const uint32_t* cnt, uint64_t slots, void* scratch, double* rho, cudaStream_t st) {
    switch (order) {
        case 1: run_sorted<1>(g, p, quantity, qscale, off, cnt, slots, scratch, rho, st); break;
        case 2: run_sorted<2>(g, p, quantity, qscale, off, cnt, slots, scratch, rho, st); break;
        case 3: run_sorted<3>(g, p, quantity, qscale, off, cnt, slots, scratch, rho, st); break;
        default: throw Status{PICGPU_EINVAL, "deposit_density: shape order must be 1, 2 or 3"};
    }
}

void launch_deposit_density_merge(int order, const GridD& g, const CSoa& p, const double* quantity, double qscale,
                                  const uint32_t* rank, const uint32_t* off, const uint32_t* cnt, uint64_t slots,
                                  void* scratch, double* rho, cudaStream_t st) {
    switch (order) {
        case 1: run_merge<1>(g, p, quantity, qscale, rank, off, cnt, slots, scratch, rho, st); break;
        case 2: run_merge<2>(g, p, quantity, qscale, rank, off, cnt, slots, scratch, rho, st); break;
        case 3: run_merge<3>(g, p, quantity, qscale, rank, off, cnt, slots, scratch, rho, st); break;
        default: throw Status{PICGPU_EINVAL, "deposit_density: shape order must be 1, 2 or 3"};
    }
}

}  // namespace picgpu

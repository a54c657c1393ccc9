// radix_sort.cu -- hand-written stable LSD radix sort of (cell key, index)
// pairs and the u32 -> u64 exclusive scan: the counting sort behind
// gpma_build / global_sort (proj/include/pic/gpma.hpp:379-402: stable counting
// sort of the particles by cell; sort_policy.hpp:83-85) and behind every
// layout (Gpma::layout, gpma.hpp:269-302: bin offsets = exclusive scan of the
// capacities).
//
// Sort (one kernel launch per 8-bit digit, "onesweep" structure):
//  * k_rs_hist: ONE read of the keys builds the digit histograms of every
//    pass (shared-memory counters per CTA, one global atomic per digit per CTA);
//    k_rs_digit_scan turns them into the global base of each digit per pass.
//  * k_rs_pass: a CTA takes the next tile of 4096 keys (dynamic tile ids, so
//    every tile's predecessors are already running: the look-back always
//    makes progress), ranks them stably inside the tile (warp by warp, item
//    by item in index order: __match_any_sync groups the lanes of one digit,
//    the group's leader bumps the warp's shared counter), publishes its 256
//    digit counts and resolves their exclusive prefix over the previous
//    tiles with a decoupled look-back (per digit one 64-bit status word per
//    tile: flag | count), scatters the tile into shared memory in digit
//    order and writes it out -- runs of one digit land on consecutive
//    global addresses.
//  Stability: tile t holds keys [4096 t, 4096 t + 4096); inside a warp items
//  are ranked in index order (item j of lane l is key base + 32 j + l, j
//  outer), warps are prefix-summed in index order, tiles in tile order.
//  Pass 0 takes its values as the identity (no value array read).
//
// Traffic per pass: 8 B read + 8 B written per key (+4 B read of the keys
// once for the histograms); HBM-bound, no library kernels.
#include <algorithm>

#include "kernels.hpp"
#include "store.hpp"

namespace picgpu {

namespace {

constexpr int RS_THREADS = 256;
constexpr int RS_WARPS = RS_THREADS / 32;
constexpr int RS_ITEMS = 16;                      // keys per thread
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;    // 4096 keys per tile
constexpr int RS_RADIX = 256;
constexpr int RS_MAX_PASSES = 4;
constexpr unsigned long long RS_FLAG_AGG = 1ull << 62;
constexpr unsigned long long RS_FLAG_PFX = 2ull << 62;
constexpr unsigned long long RS_VALUE = (1ull << 62) - 1;

__global__ void __launch_bounds__(RS_THREADS) k_rs_hist(const uint32_t* __restrict__ keys, uint64_t n, int passes,
                                                        uint32_t* __restrict__ ghist) {
    __shared__ uint32_t h[RS_MAX_PASSES][RS_RADIX];
    for (int i = threadIdx.x; i < RS_MAX_PASSES * RS_RADIX; i += RS_THREADS) (&h[0][0])[i] = 0;
    __syncthreads();
    const uint64_t stride = (uint64_t)gridDim.x * RS_THREADS * 4;
    for (uint64_t b = (uint64_t)blockIdx.x * RS_THREADS * 4; b < n; b += stride) {
        const uint64_t i0 = b + (uint64_t)threadIdx.x * 4;
        if (i0 + 3 < n && (reinterpret_cast<uintptr_t>(keys + i0) & 15) == 0) {
            const uint4 k = *reinterpret_cast<const uint4*>(keys + i0);
            const uint32_t kk[4] = {k.x, k.y, k.z, k.w};
#pragma unroll
            for (int u = 0; u < 4; ++u)
                for (int p = 0; p < passes; ++p) atomicAdd(&h[p][(kk[u] >> (8 * p)) & 255u], 1u);
        } else {
            for (uint64_t i = i0; i < i0 + 4 && i < n; ++i) {
                const uint32_t k = keys[i];
                for (int p = 0; p < passes; ++p) atomicAdd(&h[p][(k >> (8 * p)) & 255u], 1u);
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * RS_RADIX; i += RS_THREADS) {
        const uint32_t v = (&h[0][0])[i];
        if (v) atomicAdd(&ghist[i], v);
    }
}

// ghist[p][d] counts -> dbase[p][d] exclusive prefix over d (one CTA).
__global__ void __launch_bounds__(RS_RADIX) k_rs_digit_scan(const uint32_t* __restrict__ ghist, int passes,
                                                            unsigned long long* __restrict__ dbase) {
    __shared__ unsigned long long s[RS_RADIX];
    for (int p = 0; p < passes; ++p) {
        const unsigned long long v = ghist[p * RS_RADIX + threadIdx.x];
        s[threadIdx.x] = v;
        __syncthreads();
        for (int o = 1; o < RS_RADIX; o <<= 1) {
            const unsigned long long t = threadIdx.x >= o ? s[threadIdx.x - o] : 0ull;
            __syncthreads();
            s[threadIdx.x] += t;
            __syncthreads();
        }
        dbase[p * RS_RADIX + threadIdx.x] = s[threadIdx.x] - v;
        __syncthreads();
    }
}

struct RsShared {
    uint32_t wcnt[RS_WARPS][RS_RADIX];  // per-warp digit counts -> per-warp exclusive prefix
    uint32_t loc[RS_RADIX];             // tile-local digit offsets
    uint32_t wsum[RS_WARPS];            // digit-count totals of each warp's 32 digits
    unsigned long long gbase[RS_RADIX]; // global position of the tile's first key of digit d
    uint32_t k[RS_TILE];                // tile keys in digit order
    uint32_t v[RS_TILE];                // tile values in digit order
    uint32_t tile;
};

template <bool IOTA>
__global__ void __launch_bounds__(RS_THREADS) k_rs_pass(const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                        uint32_t* __restrict__ kout, uint32_t* __restrict__ vout,
                                                        uint64_t n, int shift, const unsigned long long* __restrict__ dbase,
                                                        unsigned long long* status, uint32_t* tile_counter) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    RsShared& S = *reinterpret_cast<RsShared*>(smem_raw);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < RS_WARPS * RS_RADIX; i += RS_THREADS) (&S.wcnt[0][0])[i] = 0;
    if (threadIdx.x == 0) S.tile = atomicAdd(tile_counter, 1u);
    __syncthreads();
    const uint32_t tile = S.tile;
    const uint64_t base = (uint64_t)tile * RS_TILE + (uint64_t)warp * (32 * RS_ITEMS);

    uint32_t key[RS_ITEMS], val[RS_ITEMS], rank[RS_ITEMS];
#pragma unroll
    for (int j = 0; j < RS_ITEMS; ++j) {
        const uint64_t i = base + (uint64_t)j * 32 + lane;
        const bool ok = i < n;
        key[j] = ok ? kin[i] : 0xffffffffu;
        val[j] = ok ? (IOTA ? (uint32_t)i : vin[i]) : 0u;
    }
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int j = 0; j < RS_ITEMS; ++j) {
        const uint64_t i = base + (uint64_t)j * 32 + lane;
        // out-of-range lanes get a private pseudo-digit (256 + lane): they match nobody
        const uint32_t d = i < n ? (key[j] >> shift) & 255u : 256u + lane;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const int leader = __ffs(peers) - 1;
        uint32_t old = 0;
        if (lane == leader && d < RS_RADIX) {
            old = S.wcnt[warp][d];
            S.wcnt[warp][d] = old + __popc(peers);
        }
        old = __shfl_sync(0xffffffffu, old, leader);
        rank[j] = old + __popc(peers & lt);
        __syncwarp();
    }
    __syncthreads();
    // per digit: exclusive prefix over warps, tile count; publish the aggregate
    const int d = threadIdx.x;  // RS_THREADS == RS_RADIX
    uint32_t cnt = 0;
#pragma unroll
    for (int w = 0; w < RS_WARPS; ++w) {
        const uint32_t c = S.wcnt[w][d];
        S.wcnt[w][d] = cnt;
        cnt += c;
    }
    unsigned long long* my = status + (uint64_t)tile * RS_RADIX + d;
    if (tile == 0) {
        atomicExch(my, RS_FLAG_PFX | cnt);
        S.gbase[d] = dbase[d];
    } else {
        atomicExch(my, RS_FLAG_AGG | cnt);
        unsigned long long excl = 0;
        for (int64_t p = (int64_t)tile - 1; p >= 0; --p) {
            const volatile unsigned long long* sp = status + (uint64_t)p * RS_RADIX + d;
            unsigned long long s;
            do {
                s = *sp;
            } while ((s & (RS_FLAG_AGG | RS_FLAG_PFX)) == 0);
            excl += s & RS_VALUE;
            if (s & RS_FLAG_PFX) break;
        }
        atomicExch(my, RS_FLAG_PFX | (excl + cnt));
        S.gbase[d] = dbase[d] + excl;
    }
    // tile-local digit offsets: exclusive scan of the 256 counts (warp scans + warp carries)
    {
        uint32_t x = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) S.wsum[warp] = x;
        __syncthreads();
        uint32_t carry = 0;
        for (int w = 0; w < warp; ++w) carry += S.wsum[w];
        S.loc[d] = carry + x - cnt;
    }
    __syncthreads();
    // scatter into shared memory in digit order
#pragma unroll
    for (int j = 0; j < RS_ITEMS; ++j) {
        const uint64_t i = base + (uint64_t)j * 32 + lane;
        if (i < n) {
            const uint32_t dd = (key[j] >> shift) & 255u;
            const uint32_t pos = S.loc[dd] + S.wcnt[warp][dd] + rank[j];
            S.k[pos] = key[j];
            S.v[pos] = val[j];
        }
    }
    __syncthreads();
    const uint64_t t0 = (uint64_t)tile * RS_TILE;
    const uint32_t valid = (uint32_t)(n - t0 < (uint64_t)RS_TILE ? n - t0 : (uint64_t)RS_TILE);
    for (uint32_t p = threadIdx.x; p < valid; p += RS_THREADS) {
        const uint32_t k = S.k[p];
        const uint32_t dd = (k >> shift) & 255u;
        const unsigned long long g = S.gbase[dd] + (p - S.loc[dd]);
        kout[g] = k;
        vout[g] = S.v[p];
    }
}

// ---- exclusive scan u32 -> u64 (three phases; n = ncells + 1 <= 2^32)
constexpr int SC_THREADS = 256;
constexpr int SC_ITEMS = 16;
constexpr int SC_TILE = SC_THREADS * SC_ITEMS;

__device__ __forceinline__ unsigned long long block_excl_scan(unsigned long long x, unsigned long long* sw,
                                                              unsigned long long& total) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) sw[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        unsigned long long w = lane < SC_THREADS / 32 ? sw[lane] : 0ull;
#pragma unroll
        for (int o = 1; o < SC_THREADS / 32; o <<= 1) {
            const unsigned long long y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < SC_THREADS / 32) sw[lane] = w;
    }
    __syncthreads();
    const unsigned long long carry = warp ? sw[warp - 1] : 0ull;
    total = sw[SC_THREADS / 32 - 1];
    __syncthreads();
    return carry + inc - x;
}

__global__ void __launch_bounds__(SC_THREADS) k_scan_tiles(const uint32_t* __restrict__ in, uint64_t n,
                                                           unsigned long long* __restrict__ tsum) {
    __shared__ unsigned long long sw[SC_THREADS / 32];
    const uint64_t b = (uint64_t)blockIdx.x * SC_TILE + (uint64_t)threadIdx.x * SC_ITEMS;
    unsigned long long s = 0;
#pragma unroll
    for (int j = 0; j < SC_ITEMS; ++j)
        if (b + j < n) s += in[b + j];
    unsigned long long total;
    block_excl_scan(s, sw, total);
    if (threadIdx.x == 0) tsum[blockIdx.x] = total;
}

// exclusive scan of the tile sums in place (one CTA, sequential over chunks)
__global__ void __launch_bounds__(SC_THREADS) k_scan_sums(unsigned long long* tsum, uint64_t ntiles) {
    __shared__ unsigned long long sw[SC_THREADS / 32];
    unsigned long long carry = 0;
    for (uint64_t b = 0; b < ntiles; b += SC_THREADS) {
        const uint64_t i = b + threadIdx.x;
        const unsigned long long v = i < ntiles ? tsum[i] : 0ull;
        unsigned long long total;
        const unsigned long long e = block_excl_scan(v, sw, total);
        if (i < ntiles) tsum[i] = carry + e;
        carry += total;
    }
}

__global__ void __launch_bounds__(SC_THREADS) k_scan_apply(const uint32_t* __restrict__ in, uint64_t n,
                                                           const unsigned long long* __restrict__ tsum,
                                                           unsigned long long* __restrict__ out) {
    __shared__ unsigned long long sw[SC_THREADS / 32];
    const uint64_t b = (uint64_t)blockIdx.x * SC_TILE + (uint64_t)threadIdx.x * SC_ITEMS;
    uint32_t v[SC_ITEMS];
    unsigned long long s = 0;
#pragma unroll
    for (int j = 0; j < SC_ITEMS; ++j) {
        v[j] = b + j < n ? in[b + j] : 0u;
        s += v[j];
    }
    unsigned long long total;
    unsigned long long run = tsum[blockIdx.x] + block_excl_scan(s, sw, total);
#pragma unroll
    for (int j = 0; j < SC_ITEMS; ++j)
        if (b + j < n) {
            out[b + j] = run;
            run += v[j];
        }
}

}  // namespace

void exclusive_sum_u32_to_u64(const uint32_t* in, unsigned long long* out, size_t n, DevBuf& tmp, cudaStream_t st) {
    if (!n) return;
    const uint64_t tiles = (n + SC_TILE - 1) / SC_TILE;
    tmp.ensure(tiles * 8);
    unsigned long long* tsum = tmp.as<unsigned long long>();
    k_scan_tiles<<<(unsigned)tiles, SC_THREADS, 0, st>>>(in, n, tsum);
    k_scan_sums<<<1, SC_THREADS, 0, st>>>(tsum, tiles);
    k_scan_apply<<<(unsigned)tiles, SC_THREADS, 0, st>>>(in, n, tsum, out);
    note_launch(3);
    PICGPU_CUDA_TRY(cudaGetLastError());
}

void radix_sort_pairs(const uint32_t* keys_in, uint32_t* keys_out, uint32_t* keys_tmp, const uint32_t* vals_in,
                      uint32_t* vals_out, uint32_t* vals_tmp, uint64_t n, int bits, DevBuf& tmp, cudaStream_t st) {
    const int passes = std::max(1, (bits + 7) / 8);
    if (passes > RS_MAX_PASSES) throw Status{PICGPU_ELENGTH, "radix sort: keys wider than 32 bits"};
    const uint64_t tiles = (n + RS_TILE - 1) / RS_TILE;
    if (tiles >= (1ull << 31)) throw Status{PICGPU_ELENGTH, "radix sort: too many keys"};
    if (!n) return;
    // workspace: histograms (u32), digit bases (u64), tile counters, look-back status (u64)
    const size_t hist_b = RS_MAX_PASSES * RS_RADIX * 4, dbase_b = RS_MAX_PASSES * RS_RADIX * 8, ctr_b = 256;
    const size_t status_b = tiles * RS_RADIX * 8;
    tmp.ensure(hist_b + dbase_b + ctr_b * RS_MAX_PASSES + status_b);
    char* w = tmp.as<char>();
    uint32_t* ghist = reinterpret_cast<uint32_t*>(w);
    unsigned long long* dbase = reinterpret_cast<unsigned long long*>(w + hist_b);
    uint32_t* tctr = reinterpret_cast<uint32_t*>(w + hist_b + dbase_b);
    unsigned long long* status = reinterpret_cast<unsigned long long*>(w + hist_b + dbase_b + ctr_b * RS_MAX_PASSES);
    PICGPU_CUDA_TRY(cudaMemsetAsync(w, 0, hist_b + dbase_b + ctr_b * RS_MAX_PASSES, st));
    static int hist_ctas[64] = {};
    int dev = 0;
    PICGPU_CUDA_TRY(cudaGetDevice(&dev));
    if (!hist_ctas[dev & 63]) {  // per device (one process may drive several GPUs)
        int sms = 148;
        PICGPU_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        PICGPU_CUDA_TRY(cudaFuncSetAttribute(k_rs_pass<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)sizeof(RsShared)));
        PICGPU_CUDA_TRY(cudaFuncSetAttribute(k_rs_pass<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)sizeof(RsShared)));
        hist_ctas[dev & 63] = sms * 4;
    }
    const uint64_t hctas = std::min<uint64_t>((n + RS_THREADS * 4 - 1) / (RS_THREADS * 4), (uint64_t)hist_ctas[dev & 63]);
    k_rs_hist<<<(unsigned)hctas, RS_THREADS, 0, st>>>(keys_in, n, passes, ghist);
    k_rs_digit_scan<<<1, RS_RADIX, 0, st>>>(ghist, passes, dbase);
    note_launch(2);
    // pass p writes the *_out buffers when (passes - 1 - p) is even, so the last
    // pass always lands in keys_out / vals_out; the inputs are never written
    const uint32_t* kin = keys_in;
    const uint32_t* vin = vals_in;
    for (int p = 0; p < passes; ++p) {
        const bool to_out = ((passes - 1 - p) & 1) == 0;
        uint32_t* kout = to_out ? keys_out : keys_tmp;
        uint32_t* vout = to_out ? vals_out : vals_tmp;
        PICGPU_CUDA_TRY(cudaMemsetAsync(status, 0, status_b, st));
        if (!vin)
            k_rs_pass<true><<<(unsigned)tiles, RS_THREADS, sizeof(RsShared), st>>>(
                kin, nullptr, kout, vout, n, 8 * p, dbase + p * RS_RADIX, status, tctr + p * (ctr_b / 4));
        else
            k_rs_pass<false><<<(unsigned)tiles, RS_THREADS, sizeof(RsShared), st>>>(
                kin, vin, kout, vout, n, 8 * p, dbase + p * RS_RADIX, status, tctr + p * (ctr_b / 4));
        note_launch();
        PICGPU_CUDA_TRY(cudaGetLastError());
        kin = kout;
        vin = vout;
    }
}

}  // namespace picgpu

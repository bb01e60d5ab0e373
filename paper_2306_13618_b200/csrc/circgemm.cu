// The Gaussian's spectral step without an FFT (DESIGN.md §7 "separable chain"): D_k is
// separable for the Gaussian, so F^-1 (D . F g) (the middle of the factorisation
// (4.5)-(4.6)) is the tensor power of one real symmetric circulant Csep, applied
// as one GEMM pass per axis on the box [o, o + w)^d that holds every window footprint.
//
// The passes are batched row-major fp64 GEMMs  Out_b = A_b B_b  (M = N = K = w) on the FP64
// tensor cores: mma.sync m8n8k4 f64 (SASS DMMA), 64 x 64 output tiles per 128-thread CTA
// (2 x 2 warps of 32 x 32), K in steps of 16 through a double-buffered cp.async pipeline
// (8-byte copies; a 3-stage ring of 16-byte copies when the rows are 16-byte aligned, as
// they are on the even-aligned footprint box), zero-filled at the ragged edges.  The last
// pass also zeroes the footprint box of the grid the next spread writes into (a disjoint
// buffer), which replaces a full-grid memset per half-step.
#include "common.cuh"
#include "profile.cuh"
#include "ptx.cuh"

namespace uotk {

namespace {

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
    const uint32_t d = smem_u32(dst);
    const int sz = valid ? 8 : 0;  // src-size 0: zero fill
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(valid ? src : nullptr), "r"(sz)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

struct GemmArgs {
    int M, N, K;
    const double* A;
    int64_t lda, sA;
    const double* B;
    int64_t ldb, sB;
    double* O;
    int64_t ldo, sO;
    int tiles_m, tiles_n;
    // optional side job: zero `zrows` rows of `zlen` doubles, row r at zbase + off(r)
    // (off(r) = (r / zdiv) * zs1 + (r % zdiv) * zs0)
    double* zbase;
    int64_t zrows, zlen, zdiv, zs0, zs1;
};

// BM x BN output tile per 128-thread CTA (2 x 2 warps of BM/2 x BN/2, i.e. TM x TN DMMA
// tiles of 8 x 8 per warp); K in tiles of BK through STAGES cp.async buffers.  Two
// configurations: 64 x 64 / BK 16 / 2 stages for large boxes (C4's literal 4096^2 grid:
// w = 1982), and 32 x 32 / BK 64 / 1 stage for boxes up to 64 (C3: w = 44), where the pass
// is latency-bound: 4x the CTAs, 1/4 of the DMMA chain per warp, one global round trip.
template <int BM, int BN, int BK, int STAGES, int WM = 2, int WN = 2>
__global__ void __launch_bounds__(WM * WN * 32) dgemm_rm_k(GemmArgs g) {
    constexpr int NTH = WM * WN * 32;
    constexpr int SA = BK + 4;  // A tile row stride (doubles): conflict-free fragment loads
    constexpr int SB = BN + 4;  // B tile row stride
    constexpr int TM = BM / WM / 8, TN = BN / WN / 8;  // 8 x 8 DMMA tiles per warp
    extern __shared__ __align__(16) double smem[];
    double* As = smem;                       // [STAGES][BM * SA]
    double* Bs = smem + STAGES * BM * SA;    // [STAGES][BK * SB]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp / WN, wn = warp % WN;
    const int per_batch = g.tiles_m * g.tiles_n;
    const int b = blockIdx.x / per_batch;
    const int t = blockIdx.x % per_batch;
    const int m0 = (t / g.tiles_n) * BM, n0 = (t % g.tiles_n) * BN;
    const double* A = g.A + b * g.sA;
    const double* B = g.B + b * g.sB;

    auto load = [&](int stage, int k0) {
        double* as = As + stage * BM * SA;
        double* bs = Bs + stage * BK * SB;
        for (int e = tid; e < BM * BK; e += NTH) {
            const int r = e / BK, c = e % BK;
            const bool v = m0 + r < g.M && k0 + c < g.K;
            cp_async8(&as[r * SA + c], A + (int64_t)(m0 + r) * g.lda + (k0 + c), v);
        }
        for (int e = tid; e < BK * BN; e += NTH) {
            const int r = e / BN, c = e % BN;
            const bool v = k0 + r < g.K && n0 + c < g.N;
            cp_async8(&bs[r * SB + c], B + (int64_t)(k0 + r) * g.ldb + (n0 + c), v);
        }
        cp_async_commit();
    };
    const int nk = (g.K + BK - 1) / BK;
    load(0, 0);

    // side job while the first tiles are in flight (an independent buffer): this CTA's
    // share of the rows to zero
    if (g.zbase) {
        const int64_t nblk = (int64_t)gridDim.x;
        const int64_t r0 = g.zrows * blockIdx.x / nblk, r1 = g.zrows * (blockIdx.x + 1) / nblk;
        for (int64_t r = r0; r < r1; ++r) {
            double* row = g.zbase + (r / g.zdiv) * g.zs1 + (r % g.zdiv) * g.zs0;
            for (int64_t c = tid; c < g.zlen; c += NTH) row[c] = 0.0;
        }
    }

    double acc[TM][TN][2];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (int kt = 0; kt < nk; ++kt) {
        const int st = STAGES == 1 ? 0 : kt & 1;
        if (STAGES > 1 && kt + 1 < nk) {
            load(st ^ 1, (kt + 1) * BK);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        const double* as = As + st * BM * SA;
        const double* bs = Bs + st * BK * SB;
        const int kmax = min(BK, g.K - kt * BK);  // skip the zero-filled k-steps of the last tile
        for (int kk = 0; kk < kmax; kk += 4) {
            double a[TM], bf[TN];
#pragma unroll
            for (int i = 0; i < TM; ++i) a[i] = as[(wm * (BM / WM) + i * 8 + (lane >> 2)) * SA + kk + (lane & 3)];
#pragma unroll
            for (int j = 0; j < TN; ++j) bf[j] = bs[(kk + (lane & 3)) * SB + wn * (BN / WN) + j * 8 + (lane >> 2)];
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], bf[j]);
        }
        __syncthreads();
        if (STAGES == 1 && kt + 1 < nk) load(0, (kt + 1) * BK);
    }
    double* O = g.O + b * g.sO;
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int r = m0 + wm * (BM / WM) + i * 8 + (lane >> 2);
        if (r >= g.M) continue;
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            const int c = n0 + wn * (BN / WN) + j * 8 + 2 * (lane & 3);
            if (c < g.N) O[(int64_t)r * g.ldo + c] = acc[i][j][0];
            if (c + 1 < g.N) O[(int64_t)r * g.ldo + c + 1] = acc[i][j][1];
        }
    }
}

// Large boxes with 16-byte-aligned rows (even box origin, leading dimensions and sizes —
// the box is even-aligned by choose_params): the same warp tiling, operands streamed by
// 16-byte cp.async through a 3-stage ring (two tiles in flight while one is computed).
__device__ __forceinline__ void cp_async16(double* dst, const double* src, bool valid) {
    const uint32_t d = smem_u32(dst);
    const int sz = valid ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(valid ? src : nullptr), "r"(sz)
                 : "memory");
}
template <int BM, int BN, int BK, int WM = 2, int WN = 2>
__global__ void __launch_bounds__(WM * WN * 32) dgemm_v16_k(GemmArgs g) {
    constexpr int NTH = WM * WN * 32;
    constexpr int ST = 3;
    constexpr int SA = BK + 4;
    constexpr int SB = BN + 4;
    constexpr int TM = BM / WM / 8, TN = BN / WN / 8;
    extern __shared__ __align__(16) double smem[];
    double* As = smem;                  // [ST][BM * SA]
    double* Bs = smem + ST * BM * SA;   // [ST][BK * SB]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp / WN, wn = warp % WN;
    const int per_batch = g.tiles_m * g.tiles_n;
    const int b = blockIdx.x / per_batch;
    const int t = blockIdx.x % per_batch;
    const int m0 = (t / g.tiles_n) * BM, n0 = (t % g.tiles_n) * BN;
    const double* A = g.A + b * g.sA;
    const double* B = g.B + b * g.sB;
    const int nk = (g.K + BK - 1) / BK;
    auto load = [&](int stage, int kt) {
        if (kt < nk) {
            const int k0 = kt * BK;
            double* as = As + stage * BM * SA;
            double* bs = Bs + stage * BK * SB;
            for (int e = tid; e < BM * BK / 2; e += NTH) {
                const int r = e / (BK / 2), c = 2 * (e % (BK / 2));
                const bool v = m0 + r < g.M && k0 + c < g.K;
                cp_async16(&as[r * SA + c], A + (int64_t)(m0 + r) * g.lda + (k0 + c), v);
            }
            for (int e = tid; e < BK * BN / 2; e += NTH) {
                const int r = e / (BN / 2), c = 2 * (e % (BN / 2));
                const bool v = k0 + r < g.K && n0 + c < g.N;
                cp_async16(&bs[r * SB + c], B + (int64_t)(k0 + r) * g.ldb + (n0 + c), v);
            }
        }
        cp_async_commit();  // (an empty group past the last tile keeps the wait counts uniform)
    };
    load(0, 0);
    load(1, 1);
    if (g.zbase) {
        const int64_t nblk = (int64_t)gridDim.x;
        const int64_t r0 = g.zrows * blockIdx.x / nblk, r1 = g.zrows * (blockIdx.x + 1) / nblk;
        for (int64_t r = r0; r < r1; ++r) {
            double* row = g.zbase + (r / g.zdiv) * g.zs1 + (r % g.zdiv) * g.zs0;
            for (int64_t c = tid; c < g.zlen; c += NTH) row[c] = 0.0;
        }
    }
    double acc[TM][TN][2];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    for (int kt = 0; kt < nk; ++kt) {
        cp_async_wait<1>();  // tile kt has landed (tile kt+1 may still be in flight)
        __syncthreads();     // ... for every thread; and everyone is done with tile kt-1's stage
        load((kt + 2) % ST, kt + 2);
        const double* as = As + (kt % ST) * BM * SA;
        const double* bs = Bs + (kt % ST) * BK * SB;
        const int kmax = min(BK, g.K - kt * BK);
        for (int kk = 0; kk < kmax; kk += 4) {
            double a[TM], bf[TN];
#pragma unroll
            for (int i = 0; i < TM; ++i) a[i] = as[(wm * (BM / WM) + i * 8 + (lane >> 2)) * SA + kk + (lane & 3)];
#pragma unroll
            for (int j = 0; j < TN; ++j) bf[j] = bs[(kk + (lane & 3)) * SB + wn * (BN / WN) + j * 8 + (lane >> 2)];
#pragma unroll
            for (int i = 0; i < TM; ++i)
#pragma unroll
                for (int j = 0; j < TN; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], bf[j]);
        }
    }
    double* O = g.O + b * g.sO;
#pragma unroll
    for (int i = 0; i < TM; ++i) {
        const int r = m0 + wm * (BM / WM) + i * 8 + (lane >> 2);
        if (r >= g.M) continue;
#pragma unroll
        for (int j = 0; j < TN; ++j) {
            const int c = n0 + wn * (BN / WN) + j * 8 + 2 * (lane & 3);
            if (c < g.N) O[(int64_t)r * g.ldo + c] = acc[i][j][0];
            if (c + 1 < g.N) O[(int64_t)r * g.ldo + c + 1] = acc[i][j][1];
        }
    }
}

template <int BM, int BN, int BK, int WM = 2, int WN = 2>
void launch_gemm_v16(GemmArgs g, int batch, cudaStream_t s) {
    g.tiles_m = (g.M + BM - 1) / BM;
    g.tiles_n = (g.N + BN - 1) / BN;
    const int64_t blocks = (int64_t)g.tiles_m * g.tiles_n * batch;
    const int smem = 3 * (BM * (BK + 4) + BK * (BN + 4)) * (int)sizeof(double);
    set_smem_attr((const void*)dgemm_v16_k<BM, BN, BK, WM, WN>, smem);
    dgemm_v16_k<BM, BN, BK, WM, WN><<<(unsigned)blocks, WM * WN * 32, smem, s>>>(g);
    UOTK_LAUNCHED();
}

template <int BM, int BN, int BK, int STAGES, int WM = 2, int WN = 2>
void launch_gemm(GemmArgs g, int batch, cudaStream_t s) {
    g.tiles_m = (g.M + BM - 1) / BM;
    g.tiles_n = (g.N + BN - 1) / BN;
    const int64_t blocks = (int64_t)g.tiles_m * g.tiles_n * batch;
    const int smem = (STAGES * BM * (BK + 4) + STAGES * BK * (BN + 4)) * (int)sizeof(double);
    set_smem_attr((const void*)dgemm_rm_k<BM, BN, BK, STAGES, WM, WN>, smem);
    dgemm_rm_k<BM, BN, BK, STAGES, WM, WN><<<(unsigned)blocks, WM * WN * 32, smem, s>>>(g);
    UOTK_LAUNCHED();
}

// Out_b = A_b B_b for b < batch (row-major, strides in doubles)
void gemm(int M, int N, int K, const double* A, int64_t lda, int64_t sA, const double* B, int64_t ldb, int64_t sB,
          double* O, int64_t ldo, int64_t sO, int batch, cudaStream_t s, GemmArgs zero = GemmArgs{}) {
    GemmArgs g = zero;
    g.M = M;
    g.N = N;
    g.K = K;
    g.A = A;
    g.lda = lda;
    g.sA = sA;
    g.B = B;
    g.ldb = ldb;
    g.sB = sB;
    g.O = O;
    g.ldo = ldo;
    g.sO = sO;
    const int64_t tiles64 = (int64_t)((M + 63) / 64) * ((N + 63) / 64) * batch;
    if (K <= 64 && M <= 64) launch_gemm<32, 32, 64, 1>(g, batch, s);       // C3 (w = 44)
    else if (tiles64 < 2 * 148) launch_gemm<32, 32, 32, 2>(g, batch, s);  // few tiles (C4 auto, w = 164)
    // mid-size boxes (MMD^2 / C5 at 140^3, w = 86): 32 x 32 tiles, BK = 32, two stages
    // (61 -> 40 us per chain against the 64 x 64 tiles below; a full-K 32 x 32 x 64 tile 43 us)
    else if (K <= 128 && M <= 128) launch_gemm<32, 32, 32, 2>(g, batch, s);
    else {
        // large boxes (C4 at 4096^2, w = 1982): 16-byte 3-stage operand ring when every row
        // start is 16-byte aligned, else the 8-byte 2-stage kernel (128 x 128 tiles with 8
        // warps measured 1.44 vs 1.24 ms per chain)
        const bool even = ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15) == 0 &&
                          ((lda | sA | ldb | sB | (int64_t)M | (int64_t)N | (int64_t)K) & 1) == 0;
        static const bool v16_env = [] {
            const char* e = getenv("UOTK_GEMM_V16");
            return !(e && e[0] == '0');
        }();
        // (64 x 64 x 32 and 128 x 64 x 16 three-stage variants measured 1.38 / 1.35 ms)
        if (even && v16_env) launch_gemm_v16<64, 64, 16>(g, batch, s);
        else launch_gemm<64, 64, 16, 2>(g, batch, s);
    }
}

}  // namespace

void comm_allreduce(double* buf, size_t count, int op_max_min_sum, void* comm, cudaStream_t s);  // comm.cu
void comm_reduce_scatter(const double* in, double* out, size_t count, void* comm, cudaStream_t s);
void comm_all_gather(const double* in, double* out, size_t count, void* comm, cudaStream_t s);
int comm_nranks(void* comm);
int comm_rank(void* comm);

namespace {
// d = 2, distributed pass: spare[(o + x) n + o + y] = all[(y / wb) w wb + x wb + y % wb]
__global__ void unpack_cols_k(const double* __restrict__ all, int w, int wb, int n, int o,
                              double* __restrict__ spare) {
    const int64_t total = (int64_t)w * w;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(i / w), y = (int)(i % w);
        spare[(int64_t)(o + x) * n + o + y] = all[(int64_t)(y / wb) * w * wb + (int64_t)x * wb + y % wb];
    }
}
}  // namespace

static bool dist_chain_enabled();
static int dist_chain_mode();
// the chain runs slab-distributed (reduce-scatter / middle pass on 1/P / all-gather)
static bool chain_distributed(void* comm) {
    return comm && dist_chain_enabled() && (comm_nranks(comm) > 1 || dist_chain_mode() == 2);
}

// doubles of the chain's work buffer
size_t separable_work_elems(const FastParams& fp, void* comm) {
    const size_t w = fp.box_w;
    const int P = comm_nranks(comm);
    if (fp.d == 1) return w;
    if (!chain_distributed(comm)) return fp.d == 2 ? w * w : w * w * w;
    if (fp.d == 2) {
        const size_t wb = (w + P - 1) / P;
        return (2 * (size_t)P + 2) * w * wb;
    }
    const size_t xb = (w + P - 1) / P;
    return ((size_t)P + 2) * xb * w * w;
}

// UOTK_DIST_CHAIN: 0 = one all-reduce of the first pass's box instead of the slab split;
// 2 = the slab split even on a 1-rank communicator (tests the reduce-scatter / all-gather
// calls of a real NCCL communicator on one GPU)
static int dist_chain_mode() {
    static const int mode = [] {
        const char* e = getenv("UOTK_DIST_CHAIN");
        return e ? atoi(e) : 1;
    }();
    return mode;
}
static bool dist_chain_enabled() { return dist_chain_mode() != 0; }

// g' = (Csep x ... x Csep) g on the footprint box (spread grid g: zero outside the box).
// Returns the buffer holding g' at the box positions (`spare`, n_g^d doubles).  `work`
// holds the compact intermediate (w^d doubles).  With several ranks every rank spread
// its own sources and the first pass's compact output is summed over ranks (the chain is
// linear).  zero_next (optional): a grid that is zero outside the box; its box is zeroed
// by the last pass (the next spread's target).
double* separable_chain_dmma(const FastParams& fp, const double* Csep, double* grid, double* spare, double* work,
                             double* zero_next, cudaStream_t s, void* comm) {
    const int n = fp.ng, o = fp.box_lo, w = fp.box_w, d = fp.d;
    const int64_t n2 = (int64_t)n * n, w2 = (int64_t)w * w;
    const double* Cb = Csep + (int64_t)o * n + o;  // the box block of Csep (symmetric)
    GemmArgs z{};
    if (zero_next) {
        z.zbase = zero_next + (d == 3 ? o * n2 : 0) + (d >= 2 ? (int64_t)o * n : 0) + o;
        z.zlen = w;
        z.zrows = d == 1 ? 1 : (d == 2 ? w : w2);
        z.zdiv = d == 3 ? w : 1 << 30;
        z.zs0 = d == 3 ? n : (d == 2 ? n : 0);
        z.zs1 = d == 3 ? n2 : 0;
    }
    ProfScope ps_(kProfFft, s);
    if (d == 1) {  // out[z] = sum_z' C[z][z'] g[z']   (N = 1 column)
        gemm(w, 1, w, Cb, n, 0, grid + o, 1, 0, spare + o, 1, 0, 1, s, z);
        if (comm) comm_allreduce(spare + o, (size_t)w, 0, comm, s);
        return spare;
    }
    const int P = comm_nranks(comm);
    const bool dist = chain_distributed(comm);
    if (d == 2 && dist) {
        // slab-distributed: the y-pass of each rank's own spread, written as
        // P column blocks of width wb; a reduce-scatter gives rank r the global block r; the
        // x-pass of that block only (1/P of the work); an all-gather of the output blocks
        const int r = comm_rank(comm);
        const int wb = (w + P - 1) / P;
        const int64_t blk = (int64_t)w * wb;
        double* t1 = work;                 // P x (w x wb)
        double* t1r = t1 + P * blk;        // w x wb
        double* orr = t1r + blk;           // w x wb
        double* oall = orr + blk;          // P x (w x wb)
        UOTK_CUDA(cudaMemsetAsync(t1, 0, P * blk * sizeof(double), s));
        for (int b = 0; b < P; ++b) {
            const int nb = std::min(wb, w - b * wb);
            if (nb > 0) gemm(w, nb, w, grid + (int64_t)o * n + o, n, 0, Cb + b * wb, n, 0, t1 + b * blk, wb, 0, 1, s);
        }
        comm_reduce_scatter(t1, t1r, (size_t)blk, comm, s);
        const int nr = std::min(wb, w - r * wb);
        if (nr > 0) gemm(w, nr, w, Cb, n, 0, t1r, wb, 0, orr, wb, 0, 1, s, z);
        else if (zero_next) gemm(1, 1, 1, Cb, n, 0, Cb, n, 0, orr, wb, 0, 1, s, z);  // the side job alone
        comm_all_gather(orr, oall, (size_t)blk, comm, s);
        unpack_cols_k<<<(int)std::min<int64_t>(1184, ((int64_t)w * w + 255) / 256), 256, 0, s>>>(oall, w, wb, n, o,
                                                                                               spare);
        UOTK_LAUNCHED();
        return spare;
    }
    if (d == 3 && dist && (int64_t)P * ((w + P - 1) / P) * w2 <= n2 * n) {
        // slab-distributed: the z-pass of each rank's own spread (all x-planes), a
        // reduce-scatter of x-plane blocks, the y-pass of rank r's planes only, an all-gather
        // of those planes, the x-pass (replicated).  T1 (P xb planes) sits compact in spare (its
        // capacity is >= n^3 doubles, checked above)
        const int r = comm_rank(comm);
        const int xb = (w + P - 1) / P;
        const int64_t blk = (int64_t)xb * w2;
        double* t1r = work;               // xb planes
        double* t2r = t1r + blk;          // xb planes
        double* t2 = t2r + blk;           // P xb planes
        if ((int64_t)P * xb > w) UOTK_CUDA(cudaMemsetAsync(spare + w * w2, 0, ((int64_t)P * xb - w) * w2 * sizeof(double), s));
        gemm(w, w, w, grid + o * n2 + (int64_t)o * n + o, n, n2, Cb, n, 0, spare, w, w2, w, s);
        comm_reduce_scatter(spare, t1r, (size_t)blk, comm, s);
        const int nx = std::max(0, std::min(xb, w - r * xb));
        if (nx > 0) gemm(w, w, w, Cb, n, 0, t1r, w, w2, t2r, w, w2, nx, s);
        comm_all_gather(t2r, t2, (size_t)blk, comm, s);
        gemm(w, w, w, Cb, n, 0, t2, w2, w, spare + o * n2 + (int64_t)o * n + o, n2, n, w, s, z);
        return spare;
    }
    if (d == 2) {
        // y: T1[x][y] = sum_y' g[o+x][o+y'] C[o+y'][o+y]
        gemm(w, w, w, grid + (int64_t)o * n + o, n, 0, Cb, n, 0, work, w, 0, 1, s);
        if (comm) comm_allreduce(work, (size_t)w2, 0, comm, s);
        // x: out[o+x][o+y] = sum_x' C[o+x][o+x'] T1[x'][y]
        gemm(w, w, w, Cb, n, 0, work, w, 0, spare + (int64_t)o * n + o, n, 0, 1, s, z);
        return spare;
    }
    // d = 3.  z, per x: T1[x][y][z] = sum_z' g[o+x][o+y][o+z'] C[o+z'][o+z]   (T1 compact in spare)
    gemm(w, w, w, grid + o * n2 + (int64_t)o * n + o, n, n2, Cb, n, 0, spare, w, w2, w, s);
    if (comm) comm_allreduce(spare, (size_t)(w2 * w), 0, comm, s);
    // y, per x: T2[x][y][z] = sum_y' C[o+y][o+y'] T1[x][y'][z]                (T2 compact in work)
    gemm(w, w, w, Cb, n, 0, spare, w, w2, work, w, w2, w, s);
    // x, per y: out[o+x][o+y][o+z] = sum_x' C[o+x][o+x'] T2[x'][y][z]          (box positions of spare)
    gemm(w, w, w, Cb, n, 0, work, w2, w, spare + o * n2 + (int64_t)o * n + o, n2, n, w, s, z);
    return spare;
}

// MMD^2 for the Gaussian without an FFT: sum_k D_k |G_k|^2 = <g, F^-1 (D . F g)> = <g, g'>
// with g' the separable chain's output — the grid g is zero outside the footprint box, so
// the inner product runs over the box only.  part[b] = this block's partial sum (fixed
// order), reduced afterwards.
namespace {
__global__ void box_dot_k(const double* __restrict__ g, const double* __restrict__ gp, int d, int n, int o, int w,
                          int64_t total, double* __restrict__ part) {
    __shared__ double sm[256];
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t rem = i, off = 0, stride = 1;
        for (int t = 0; t < d; ++t) {
            off += (o + rem % w) * stride;
            rem /= w;
            stride *= n;
        }
        acc = fma(g[off], gp[off], acc);
    }
    sm[threadIdx.x] = acc;
    __syncthreads();
    for (int k = 128; k > 0; k >>= 1) {
        if (threadIdx.x < k) sm[threadIdx.x] += sm[threadIdx.x + k];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = sm[0];
}
}  // namespace

void box_dot(const double* g, const double* gp, const FastParams& fp, double* part, int nparts, cudaStream_t s) {
    int64_t total = 1;
    for (int t = 0; t < fp.d; ++t) total *= fp.box_w;
    box_dot_k<<<nparts, 256, 0, s>>>(g, gp, fp.d, fp.ng, fp.box_lo, fp.box_w, total, part);
    UOTK_LAUNCHED();
}

}  // namespace uotk

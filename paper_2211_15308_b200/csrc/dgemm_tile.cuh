// FP64 DMMA GEMM tile template (sm_100a), shared by libdd and tools/gemm_lab.cu.
//
//   C = A · B,  A row-major (lda), B column-major (ldb) — both K-contiguous ("TN").
//
// CTA tile BM x BN, K-step BK, WM x WN warps each owning (BM/WM) x (BN/WN) as m16n8k4 fragments
// (mma.sync.aligned.m16n8k4 .f64 -> SASS DMMA.8x8x4; tcgen05 has no f64 kind).  Operands are
// staged by a STAGES-deep cp.async (LDGSTS) ring in padded smem rows (BK+4 doubles: the
// fragment loads of a warp hit distinct bank pairs).  Split-K: gridDim.y = S CTAs of one output
// tile form a thread-block cluster (1, S, 1) (S = 1, 2, 4, 8, a template parameter).  After its
// main loop each CTA q PUSHES accumulator register r into slot [q] of CTA (r mod S)'s reduction
// buffer with st.shared::cluster (a region of its own, so pushes may land while the owner is
// still in its main loop); one cluster barrier (arrive.release / wait.acquire); each CTA then sums
// its S slots from local shared memory in fixed order q = 0..S-1 (bitwise deterministic, no
// global partials, no remote loads) and runs the epilogue on its registers r ≡ rank (mod S).
// Programmatic dependent launch: every kernel lets its dependents launch at entry
// (griddepcontrol.launch_dependents) and waits for its prerequisite grid (griddepcontrol.wait)
// only before touching data the preceding kernel may write; with `a_static` the first A stages
// (a constant operand, e.g. the sine matrix) are prefetched before that wait.
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>

namespace dd {
namespace cg = cooperative_groups;

template <int BM_, int BN_, int BK_, int WM_, int WN_, int STAGES_, int MINB_>
struct DgemmCfg {
    static constexpr int BM = BM_, BN = BN_, BK = BK_, WM = WM_, WN = WN_, STAGES = STAGES_, MINB = MINB_;
    static constexpr int THREADS = WM * WN * 32;
    static constexpr int LDS = BK + 4;
    static constexpr int TM = BM / WM, TN = BN / WN;        // warp tile
    static constexpr int MI = TM / 16, NI = TN / 8;         // fragments per warp
    static constexpr int NREG = MI * NI * 4;                // accumulators per thread
    static constexpr size_t SMEM_PIPE = size_t(STAGES) * (BM + BN) * LDS * sizeof(double);
    static constexpr size_t SMEM_RED = size_t(NREG) * THREADS * sizeof(double);
    static constexpr size_t SMEM = SMEM_PIPE > SMEM_RED ? SMEM_PIPE : SMEM_RED;
    static constexpr int CPR = BK / 2;                      // 16-byte chunks per smem row
    static constexpr int ACH = BM * CPR, BCH = BN * CPR;    // chunks per stage
    static_assert(TM % 16 == 0 && TN % 8 == 0 && BK % 4 == 0, "tile shape");
};

// Batched problem: gridDim.z = batch; slab b uses A + b*sA, B + b*sB and the epilogue gets b.
struct DgemmProblem {
    int M, N, K;                 // K multiple of BK
    const double* A; int lda;    // rows readable up to round_up(M, BM)
    const double* B; int ldb;    // columns readable up to round_up(N, BN)
    long long sA = 0, sB = 0;    // batch strides (elements)
    int batch = 1;
    const int* active = nullptr; // optional per-slab flag: slabs with active[b] == 0 are skipped
    unsigned long long* ts = nullptr;   // optional per-CTA phase timestamps (lab instrumentation)
    int a_static = 0;            // A is not written by the preceding kernel: prefetch it before griddepcontrol.wait
    const int* ntl = nullptr;    // live column tiles [count, tile ids...] of width ntl_bn (PCG: columns freeze
                                 // when converged): the tile / stream-K work is laid out over the live tiles only
    int ntl_bn = 64;             // live-tile width, a multiple of BN
    // Grouped A (tile kernel only): column tile [n0, n0+BN) multiplies A + col_group[n0] * sG —
    // every BN-column tile must lie in one group — unless *mixed != 0 (flag written on the device
    // before this launch), in which case the whole launch computes the fallback product
    // alt_A (M x alt_K, lda alt_lda) x alt_B (ldb alt_ldb) instead.
    const int* col_group = nullptr;
    int n_group = 1;                    // group ids are clamped to [0, n_group)
    long long sG = 0;
    const int* mixed = nullptr;
    const double* alt_A = nullptr; int alt_lda = 0;
    const double* alt_B = nullptr; int alt_ldb = 0;
    int alt_K = 0;
    // Parity-blocked B (tile kernel, S = 1 slabs; not with ntl / col_group): B = [[0, E], [E', 0]]
    // with the block edge at kpar (a multiple of BN and BK) — a column tile below kpar only needs
    // k in [kpar, K), one at or above it k in [0, kpar); the skipped products are exact zeros
    // (fma(0, a, acc) == acc), so the result is bitwise that of the full K loop.  0: full K.
    int kpar = 0;
};

// Programmatic dependent launch (no-ops when the launch did not opt in)
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ unsigned long long dg_gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define DG_TS(i) \
    if (g.ts && threadIdx.x == 0) g.ts[(size_t)(blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z)) * 8 + (i)] = dg_gtime()

__device__ __forceinline__ void dg_cp_async16(void* smem, const void* gmem) {
    unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void dg_cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void dg_cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dg_mma(double (&c)[4], double a0, double a1, double b) {
    asm volatile(
        "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
        : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
        : "d"(a0), "d"(a1), "d"(b));
}

// Row / column of accumulator register r of this thread within the CTA tile.
template <class C>
__device__ __forceinline__ void dg_coord(int r, int tid, int& row, int& col) {
    const int warp = tid >> 5, lane = tid & 31;
    const int wm = warp % C::WM, wn = warp / C::WM;
    const int f = r >> 2, q = r & 3;
    const int mi = f / C::NI, ni = f % C::NI;
    row = wm * C::TM + mi * 16 + (lane >> 2) + (q >> 1) * 8;
    col = wn * C::TN + ni * 8 + (lane & 3) * 2 + (q & 1);
}

// Issue the cp.async copies of one K-stage (A: BM rows, B: BN columns of BK doubles each).
template <class C>
__device__ __forceinline__ void dg_load_A(double* As, const double* A, int lda, int m0, int k0, int tid) {
#pragma unroll
    for (int j = 0; j < (C::ACH + C::THREADS - 1) / C::THREADS; j++) {
        const int c = tid + C::THREADS * j;
        if (C::ACH % C::THREADS == 0 || c < C::ACH) {
            const int row = c / C::CPR, kc = (c % C::CPR) * 2;
            dg_cp_async16(&As[row * C::LDS + kc], A + (size_t)(m0 + row) * lda + k0 + kc);
        }
    }
}
template <class C>
__device__ __forceinline__ void dg_load_B(double* Bs, const double* B, int ldb, int n0, int k0, int tid) {
#pragma unroll
    for (int j = 0; j < (C::BCH + C::THREADS - 1) / C::THREADS; j++) {
        const int c = tid + C::THREADS * j;
        if (C::BCH % C::THREADS == 0 || c < C::BCH) {
            const int row = c / C::CPR, kc = (c % C::CPR) * 2;
            dg_cp_async16(&Bs[row * C::LDS + kc], B + (size_t)(n0 + row) * ldb + k0 + kc);
        }
    }
}
template <class C>
__device__ __forceinline__ void dg_load_stage(double* As, double* Bs, const double* A, int lda, const double* B, int ldb,
                                              int m0, int n0, int k0, int tid) {
    dg_load_A<C>(As, A, lda, m0, k0, tid);
    dg_load_B<C>(Bs, B, ldb, n0, k0, tid);
}

// Shared memory of the split-K tile kernel: the pipeline ring plus (S > 1) a separate
// reduction buffer [S][ceil(NREG/S)][THREADS].
template <class C, int S>
constexpr size_t dg_tile_smem() {
    return C::SMEM_PIPE + (S > 1 ? size_t(S) * ((C::NREG + S - 1) / S) * C::THREADS * sizeof(double) : 0);
}

// Epi: functor  __device__ void operator()(int b, int row, int col, double v) const
// (b = batch index; row < M, col < N checked)
//
// Staged epilogue (tile kernel, S = 1): an Epi with `static constexpr bool kStaged = true` gets the
// CTA tile through shared memory, transposed to column-contiguous row pairs, and is called as
//   Blk k = epi.block(b);                       once per CTA (per-slab scalars)
//   epi.load(b, row, col, k, ctx);              U row pairs (row, row+1) of column col ...
//   epi.store(b, row, col, pair, k, ctx, v);    ... then their results (pair: row+1 < M)
// so that a functor whose stores may alias its loads (in-place updates) still issues U
// independent 16-byte loads per thread before the first store — the per-element form serialises
// every load behind the previous element's store.  Output addresses of a row pair are
// contiguous when the epilogue stores transposed (i = row + col * ld), as the slab passes do.
template <class Epi, class = void>
struct EpiStaged { static constexpr bool value = false; };
template <class Epi>
struct EpiStaged<Epi, decltype(void(Epi::kStaged))> { static constexpr bool value = Epi::kStaged; };
template <class C, class Epi, int S>
__global__ void __launch_bounds__(C::THREADS, C::MINB) k_dgemm_tile(DgemmProblem g, Epi epi) {
    extern __shared__ __align__(16) double smem[];
    double* As = smem;
    double* Bs = smem + C::STAGES * C::BM * C::LDS;
    pdl_launch_dependents();
    const int bz = blockIdx.z;
    const int tiles_m = (g.M + C::BM - 1) / C::BM;
    const int m0 = (blockIdx.x % tiles_m) * C::BM;
    int n0 = (blockIdx.x / tiles_m) * C::BN;
    const int split = S > 1 ? (int)blockIdx.y : 0;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wm = warp % C::WM, wn = warp / C::WM;
    const int gq = lane >> 2, tq = lane & 3;

    // prologue: constant A stages may be fetched before the prerequisite grid has finished.
    // Grouped A: the group ids and the mixed flag are written before the first PDL launch of
    // a solve (their producers are launched without PDL), so they may be read here too — unless
    // a live-tile list (written by the preceding kernel) decides which tile this CTA takes.
    const bool pre_a = g.a_static && !g.active && !(g.col_group && g.ntl);
    const double* A0 = g.A + (size_t)bz * g.sA;
    bool resolved = false;
    auto resolve_group = [&]() {
        if (g.mixed && *g.mixed) {           // uniform across the grid
            A0 = g.alt_A; g.lda = g.alt_lda; g.B = g.alt_B; g.ldb = g.alt_ldb; g.K = g.alt_K;
        } else {
            int grp = n0 < g.N ? g.col_group[n0] : 0;
            grp = grp < 0 ? 0 : (grp >= g.n_group ? g.n_group - 1 : grp);
            A0 = g.A + (size_t)grp * g.sG;
        }
        resolved = true;
    };
    if (g.col_group && !g.ntl) resolve_group();
    int nkt, kt0;
    {
        int kb = 0, ke = g.K;
        if (g.kpar) {
            if (n0 + C::BN <= g.kpar) kb = g.kpar;
            else if (n0 >= g.kpar) ke = g.kpar;
        }
        const int ktiles = (ke - kb) / C::BK;
        const int per = (ktiles + S - 1) / S;
        nkt = max(0, min(per, ktiles - split * per));
        kt0 = kb / C::BK + split * per;
    }
    if (pre_a) {
#pragma unroll
        for (int s = 0; s < C::STAGES - 1; s++)
            if (s < nkt) dg_load_A<C>(As + s * C::BM * C::LDS, A0, g.lda, m0, (kt0 + s) * C::BK, tid);
    }
    pdl_wait();
    if (g.active && !g.active[bz]) return;   // frozen slab (uniform across the cluster)
    if (g.ntl) {                             // live column tiles only (uniform across the cluster)
        const int SUB = g.ntl_bn / C::BN;
        const int nidx = blockIdx.x / tiles_m;
        if (nidx / SUB >= g.ntl[0]) {
            asm volatile("cp.async.wait_all;\n" ::);   // drain the A prefetch before leaving
            return;
        }
        n0 = g.ntl[1 + nidx / SUB] * g.ntl_bn + (nidx % SUB) * C::BN;
        if (n0 >= g.N) {                     // ragged half of the last live tile
            asm volatile("cp.async.wait_all;\n" ::);
            return;
        }
    }
    if (g.col_group && !resolved) {
        resolve_group();
        const int ktiles = g.K / C::BK;
        const int per = (ktiles + S - 1) / S;
        kt0 = split * per;
        nkt = max(0, min(per, ktiles - kt0));
    }
    DG_TS(0);
    g.A = A0;
    g.B += (size_t)bz * g.sB;

    double acc[C::MI][C::NI][4];
#pragma unroll
    for (int i = 0; i < C::MI; i++)
#pragma unroll
        for (int j = 0; j < C::NI; j++)
#pragma unroll
            for (int r = 0; r < 4; r++) acc[i][j][r] = 0.0;

#pragma unroll
    for (int s = 0; s < C::STAGES - 1; s++) {
        if (s < nkt) {
            if (!pre_a) dg_load_A<C>(As + s * C::BM * C::LDS, g.A, g.lda, m0, (kt0 + s) * C::BK, tid);
            dg_load_B<C>(Bs + s * C::BN * C::LDS, g.B, g.ldb, n0, (kt0 + s) * C::BK, tid);
        }
        dg_cp_commit();
    }
    for (int it = 0; it < nkt; it++) {
        dg_cp_wait<C::STAGES - 2>();
        __syncthreads();
        const int nk = it + C::STAGES - 1;
        if (nk < nkt)
            dg_load_stage<C>(As + (nk % C::STAGES) * C::BM * C::LDS, Bs + (nk % C::STAGES) * C::BN * C::LDS, g.A, g.lda,
                             g.B, g.ldb, m0, n0, (kt0 + nk) * C::BK, tid);
        dg_cp_commit();
        const double* as = As + (it % C::STAGES) * C::BM * C::LDS + (wm * C::TM + gq) * C::LDS + tq;
        const double* bs = Bs + (it % C::STAGES) * C::BN * C::LDS + (wn * C::TN + gq) * C::LDS + tq;
#pragma unroll
        for (int kk = 0; kk < C::BK; kk += 4) {
            double a[C::MI][2], b[C::NI];
#pragma unroll
            for (int mi = 0; mi < C::MI; mi++) {
                a[mi][0] = as[(mi * 16) * C::LDS + kk];
                a[mi][1] = as[(mi * 16 + 8) * C::LDS + kk];
            }
#pragma unroll
            for (int ni = 0; ni < C::NI; ni++) b[ni] = bs[(ni * 8) * C::LDS + kk];
#pragma unroll
            for (int mi = 0; mi < C::MI; mi++)
#pragma unroll
                for (int ni = 0; ni < C::NI; ni++) dg_mma(acc[mi][ni], a[mi][0], a[mi][1], b[ni]);
        }
    }
    dg_cp_wait<0>();
    DG_TS(1);

    if constexpr (S == 1 && EpiStaged<Epi>::value) {
        constexpr int TLD = C::BM + 2;                    // smem column stride (even: 16-byte row pairs)
        static_assert(size_t(C::BN) * TLD * sizeof(double) <= C::SMEM_PIPE, "staged epilogue tile");
        constexpr int RP = C::BM / 2, TOT = C::BN * RP, U = 4;
        __syncthreads();                                  // every warp is done with the pipeline ring
        double* Ts = smem;
#pragma unroll
        for (int mi = 0; mi < C::MI; mi++)
#pragma unroll
            for (int ni = 0; ni < C::NI; ni++)
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    int row, col;
                    dg_coord<C>((mi * C::NI + ni) * 4 + q, tid, row, col);
                    Ts[col * TLD + row] = acc[mi][ni][q];
                }
        __syncthreads();
        const auto blk = epi.block(bz);
        for (int base = 0; base < TOT; base += C::THREADS * U) {
            typename Epi::Ctx cx[U];
            int rr[U], cc[U];
            bool ok[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int e = base + u * C::THREADS + tid;
                cc[u] = e / RP;
                rr[u] = 2 * (e % RP);
                ok[u] = e < TOT && m0 + rr[u] < g.M && n0 + cc[u] < g.N;
                if (ok[u]) epi.load(bz, m0 + rr[u], n0 + cc[u], blk, cx[u]);
            }
#pragma unroll
            for (int u = 0; u < U; u++)
                if (ok[u]) {
                    const double2 v = *reinterpret_cast<const double2*>(&Ts[cc[u] * TLD + rr[u]]);
                    epi.store(bz, m0 + rr[u], n0 + cc[u], m0 + rr[u] + 1 < g.M, blk, cx[u], v);
                }
        }
    } else if constexpr (S == 1) {
#pragma unroll
        for (int mi = 0; mi < C::MI; mi++)
#pragma unroll
            for (int ni = 0; ni < C::NI; ni++)
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    int row, col;
                    dg_coord<C>((mi * C::NI + ni) * 4 + q, tid, row, col);
                    row += m0; col += n0;
                    if (row < g.M && col < g.N) epi(bz, row, col, acc[mi][ni][q]);
                }
    } else {
        // ---- split-K: push partials into the owners' reduction buffers over DSMEM, one barrier
        constexpr int JP = (C::NREG + S - 1) / S;
        double* red = smem + C::SMEM_PIPE / sizeof(double);
        const unsigned lred = static_cast<unsigned>(__cvta_generic_to_shared(red));
        unsigned rbase[S];
#pragma unroll
        for (int o = 0; o < S; o++) asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbase[o]) : "r"(lred), "r"(o));
#pragma unroll
        for (int mi = 0; mi < C::MI; mi++)
#pragma unroll
            for (int ni = 0; ni < C::NI; ni++)
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    const int r = (mi * C::NI + ni) * 4 + q;
                    const unsigned dst = rbase[r % S] + (unsigned)(((split * JP + r / S) * C::THREADS + tid) * sizeof(double));
                    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(dst), "d"(acc[mi][ni][q]) : "memory");
                }
        asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
        DG_TS(2);
        double v[JP];
#pragma unroll
        for (int j = 0; j < JP; j++) v[j] = 0.0;
#pragma unroll
        for (int q = 0; q < S; q++)
#pragma unroll
            for (int j = 0; j < JP; j++)
                if (split + j * S < C::NREG) v[j] += red[(q * JP + j) * C::THREADS + tid];
        DG_TS(3);
#pragma unroll
        for (int j = 0; j < JP; j++) {
            const int r = split + j * S;
            if (r < C::NREG) {
                int row, col;
                dg_coord<C>(r, tid, row, col);
                row += m0; col += n0;
                if (row < g.M && col < g.N) epi(bz, row, col, v[j]);
            }
        }
        DG_TS(4);
    }
}

// ----------------------------------------------------------------------------------- stream-K
// Work units = (output tile, k-tile) pairs in tile-major, k-minor order; CTA b of G takes
// units [floor(bU/G), floor((b+1)U/G)) — every SM gets the same amount of MMA work whatever
// the tile count.  A tile whose k-range is cut by CTA boundaries is produced in segments; each
// segment's CTA parks its partial accumulators in a global slot (tile-local segment index),
// and the last CTA to finish a segment of that tile (per-tile arrival counter) sums all
// segments in segment order (its own from registers) and runs the epilogue.  Fixed partition
// + fixed order = bitwise deterministic; no CTA ever waits on another.
struct StreamK {
    double* ws;       // [slots][BM*BN] partials (slot = seg_base[tile] + seg)
    int* counters;    // [tiles], zero on entry, reset by the reducing CTA
    int G;            // CTAs in the grid
};

__device__ __forceinline__ long long sk_unit_begin(int b, long long U, int G) { return (long long)b * U / G; }
// CTA whose range contains unit u
__device__ __forceinline__ int sk_cta_of(long long u, long long U, int G) {
    int b = (int)((u * G) / U);
    while (b + 1 < G && sk_unit_begin(b + 1, U, G) <= u) b++;
    while (b > 0 && sk_unit_begin(b, U, G) > u) b--;
    return b;
}

template <class C, class Epi>
__global__ void __launch_bounds__(C::THREADS, C::MINB) k_dgemm_streamk(DgemmProblem g, Epi epi, StreamK sk) {
    extern __shared__ __align__(16) double smem[];
    double* As = smem;
    double* Bs = smem + C::STAGES * C::BM * C::LDS;
    __shared__ int s_last;
    pdl_launch_dependents();
    pdl_wait();
    bool grouped = g.col_group != nullptr;
    if (grouped && g.mixed && *g.mixed) {    // a tile spans two groups: fallback product (uniform)
        g.A = g.alt_A; g.lda = g.alt_lda; g.B = g.alt_B; g.ldb = g.alt_ldb; g.K = g.alt_K;
        grouped = false;
    }

    const int tiles_m = (g.M + C::BM - 1) / C::BM;
    const int tiles = tiles_m * (g.ntl ? g.ntl[0] * (g.ntl_bn / C::BN) : (g.N + C::BN - 1) / C::BN);
    const int KT = g.K / C::BK;
    const long long U = (long long)tiles * KT;
    const int b = blockIdx.x;
    const long long u0 = sk_unit_begin(b, U, sk.G), u1 = sk_unit_begin(b + 1, U, sk.G);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int wm = warp % C::WM, wn = warp / C::WM;
    const int gq = lane >> 2, tq = lane & 3;

    long long u = u0;
    while (u < u1) {
        const int t = (int)(u / KT);
        const int ks = (int)(u % KT);
        const int ke = (int)min((long long)KT, (long long)ks + (u1 - u));
        const int m0 = (t % tiles_m) * C::BM;
        const int n0 = g.ntl ? g.ntl[1 + (t / tiles_m) / (g.ntl_bn / C::BN)] * g.ntl_bn +
                                   ((t / tiles_m) % (g.ntl_bn / C::BN)) * C::BN
                             : (t / tiles_m) * C::BN;
        const int nkt = ke - ks;
        const double* Aseg = g.A;
        if (grouped) {
            int grp = n0 < g.N ? g.col_group[n0] : 0;
            grp = grp < 0 ? 0 : (grp >= g.n_group ? g.n_group - 1 : grp);
            Aseg = g.A + (size_t)grp * g.sG;
        }

        double acc[C::MI][C::NI][4];
#pragma unroll
        for (int i = 0; i < C::MI; i++)
#pragma unroll
            for (int j = 0; j < C::NI; j++)
#pragma unroll
                for (int r = 0; r < 4; r++) acc[i][j][r] = 0.0;

        auto load_stage = [&](int stage, int kt) {
            dg_load_stage<C>(As + stage * C::BM * C::LDS, Bs + stage * C::BN * C::LDS, Aseg, g.lda, g.B, g.ldb, m0, n0,
                             kt * C::BK, tid);
        };
        __syncthreads();   // previous segment's smem reads are finished
#pragma unroll
        for (int s = 0; s < C::STAGES - 1; s++) {
            if (s < nkt) load_stage(s, ks + s);
            dg_cp_commit();
        }
        for (int it = 0; it < nkt; it++) {
            dg_cp_wait<C::STAGES - 2>();
            __syncthreads();
            const int nk = it + C::STAGES - 1;
            if (nk < nkt) load_stage(nk % C::STAGES, ks + nk);
            dg_cp_commit();
            const double* as = As + (it % C::STAGES) * C::BM * C::LDS + (wm * C::TM + gq) * C::LDS + tq;
            const double* bs = Bs + (it % C::STAGES) * C::BN * C::LDS + (wn * C::TN + gq) * C::LDS + tq;
#pragma unroll
            for (int kk = 0; kk < C::BK; kk += 4) {
                double a[C::MI][2], bb[C::NI];
#pragma unroll
                for (int mi = 0; mi < C::MI; mi++) {
                    a[mi][0] = as[(mi * 16) * C::LDS + kk];
                    a[mi][1] = as[(mi * 16 + 8) * C::LDS + kk];
                }
#pragma unroll
                for (int ni = 0; ni < C::NI; ni++) bb[ni] = bs[(ni * 8) * C::LDS + kk];
#pragma unroll
                for (int mi = 0; mi < C::MI; mi++)
#pragma unroll
                    for (int ni = 0; ni < C::NI; ni++) dg_mma(acc[mi][ni], a[mi][0], a[mi][1], bb[ni]);
            }
        }
        dg_cp_wait<0>();

        bool emit = true;
        if (!(ks == 0 && ke == KT)) {
            // segmented tile: park the partial, count arrivals, last arriver reduces
            const long long tu0 = (long long)t * KT;
            const int bfirst = sk_cta_of(tu0, U, sk.G);
            const int blast = sk_cta_of(tu0 + KT - 1, U, sk.G);
            const int nseg = blast - bfirst + 1;
            const int seg = b - bfirst;
            // slot base of tile t = Σ_{t'<t} (nseg(t') - 1) ... use a closed form: bfirst + t
            double* slot = sk.ws + ((size_t)(bfirst + t) + seg) * (C::BM * C::BN);
#pragma unroll
            for (int mi = 0; mi < C::MI; mi++)
#pragma unroll
                for (int ni = 0; ni < C::NI; ni++)
#pragma unroll
                    for (int q = 0; q < 4; q++) __stcg(&slot[((mi * C::NI + ni) * 4 + q) * C::THREADS + tid], acc[mi][ni][q]);
            __threadfence();
            __syncthreads();
            if (tid == 0) s_last = (atomicAdd(&sk.counters[t], 1) == nseg - 1);
            __syncthreads();
            emit = s_last;
            if (emit) {
                __threadfence();
                const double* base = sk.ws + (size_t)(bfirst + t) * (C::BM * C::BN);
                // segment-outer / register-inner: each segment's loads are independent and in
                // flight together; the sum order (segment 0, 1, ...) is fixed.
                double sum[C::NREG];
#pragma unroll
                for (int r = 0; r < C::NREG; r++) sum[r] = 0.0;
                for (int s2 = 0; s2 < nseg; s2++) {
                    if (s2 == seg) {
#pragma unroll
                        for (int mi = 0; mi < C::MI; mi++)
#pragma unroll
                            for (int ni = 0; ni < C::NI; ni++)
#pragma unroll
                                for (int q = 0; q < 4; q++) sum[(mi * C::NI + ni) * 4 + q] += acc[mi][ni][q];
                    } else {
                        const double* src = base + (size_t)s2 * (C::BM * C::BN) + tid;
                        double tmp[C::NREG];
#pragma unroll
                        for (int r = 0; r < C::NREG; r++) tmp[r] = __ldcg(&src[r * C::THREADS]);
#pragma unroll
                        for (int r = 0; r < C::NREG; r++) sum[r] += tmp[r];
                    }
                }
#pragma unroll
                for (int mi = 0; mi < C::MI; mi++)
#pragma unroll
                    for (int ni = 0; ni < C::NI; ni++)
#pragma unroll
                        for (int q = 0; q < 4; q++) acc[mi][ni][q] = sum[(mi * C::NI + ni) * 4 + q];
                if (tid == 0) sk.counters[t] = 0;
            }
        }
        if (emit) {
#pragma unroll
            for (int mi = 0; mi < C::MI; mi++)
#pragma unroll
                for (int ni = 0; ni < C::NI; ni++)
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        int row, col;
                        dg_coord<C>((mi * C::NI + ni) * 4 + q, tid, row, col);
                        row += m0; col += n0;
                        if (row < g.M && col < g.N) epi(0, row, col, acc[mi][ni][q]);
                    }
        }
        u += nkt;
    }
}

// Stream-K sizing: grid = resident CTAs (SMs x occupancy, capped by the unit count).
template <class C>
inline int dgemm_streamk_grid(int M, int N, int K, int num_sms, int occ) {
    const long long tiles = ((M + C::BM - 1) / C::BM) * (long long)((N + C::BN - 1) / C::BN);
    const long long U = tiles * (K / C::BK);
    long long G = (long long)num_sms * occ;
    if (G > U) G = U;
    return (int)(G < 1 ? 1 : G);
}
// workspace: slot index bfirst(t) + t + seg <= (G - 1) + (tiles - 1) + nseg <= G + 2 tiles
template <class C>
inline size_t dgemm_streamk_ws_doubles(int M, int N, int G) {
    const size_t tiles = size_t((M + C::BM - 1) / C::BM) * size_t((N + C::BN - 1) / C::BN);
    return (size_t(G) + 2 * tiles + 2) * C::BM * C::BN;
}

// PDL launch attribute (programmatic stream serialisation) for launches that follow a kernel
inline void dg_set_pdl(cudaLaunchConfig_t& cfg, cudaLaunchAttribute* at, bool pdl) {
    if (pdl) {
        at[cfg.numAttrs].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[cfg.numAttrs].val.programmaticStreamSerializationAllowed = 1;
        cfg.numAttrs++;
    }
}

template <class C, class Epi>
inline cudaError_t dgemm_launch_streamk(const DgemmProblem& g, int G, const StreamK& sk, const Epi& epi, cudaStream_t st,
                                        bool pdl = false) {
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_dgemm_streamk<C, Epi>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    if (g.M <= 0 || g.N <= 0) return cudaSuccess;
    StreamK s = sk;
    s.G = G;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G, 1, 1);
    cfg.blockDim = dim3(C::THREADS, 1, 1);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    cfg.attrs = at;
    cfg.numAttrs = 0;
    dg_set_pdl(cfg, at, pdl);
    return cudaLaunchKernelEx(&cfg, k_dgemm_streamk<C, Epi>, g, epi, s);
}

template <class C>
inline int dgemm_tiles(int M, int N) {
    return ((M + C::BM - 1) / C::BM) * ((N + C::BN - 1) / C::BN);
}

template <class C, class Epi, int S>
inline cudaError_t dgemm_launch_s(const DgemmProblem& g, const Epi& epi, cudaStream_t st, bool pdl) {
    constexpr size_t smem = dg_tile_smem<C, S>();
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_dgemm_tile<C, Epi, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        if (smem > 100 * 1024) cudaFuncSetAttribute(k_dgemm_tile<C, Epi, S>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        attr = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(dgemm_tiles<C>(g.M, g.N), S, g.batch < 1 ? 1 : g.batch);
    cfg.blockDim = dim3(C::THREADS, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    cfg.attrs = at;
    cfg.numAttrs = 0;
    if (S > 1) {
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 1;
        at[0].val.clusterDim.y = S;
        at[0].val.clusterDim.z = 1;
        cfg.numAttrs = 1;
    }
    dg_set_pdl(cfg, at, pdl);
    return cudaLaunchKernelEx(&cfg, k_dgemm_tile<C, Epi, S>, g, epi);
}

// split-K S is rounded down to a power of two (1, 2, 4, 8)
template <class C, class Epi>
inline cudaError_t dgemm_launch(const DgemmProblem& g, int splitk, const Epi& epi, cudaStream_t st, bool pdl = false) {
    if (g.M <= 0 || g.N <= 0) return cudaSuccess;
    if (splitk >= 8) return dgemm_launch_s<C, Epi, 8>(g, epi, st, pdl);
    if (splitk >= 4) return dgemm_launch_s<C, Epi, 4>(g, epi, st, pdl);
    if (splitk >= 2) return dgemm_launch_s<C, Epi, 2>(g, epi, st, pdl);
    return dgemm_launch_s<C, Epi, 1>(g, epi, st, pdl);
}

// Pick split-K S (1..8) for a tile count so that S * tiles fills the SM slots evenly.
template <class C>
inline int dgemm_pick_splitk(int M, int N, int K, int num_sms, int ctas_per_sm) {
    const int tiles = dgemm_tiles<C>(M, N);
    const int ktiles = K / C::BK;
    const int slots = num_sms * ctas_per_sm;
    int best = 1;
    double best_t = 1e30;
    for (int s = 1; s <= 8; s *= 2) {
        if (s > 1 && ktiles / s < 4) break;
        const int ctas = tiles * s;
        // time ~ (work per CTA) x (CTAs on the busiest SM) / (SM efficiency at that residency):
        // one 4-warp CTA alone keeps the DMMA pipe ~60% busy, two or more ~100% (gemm_lab).
        const double per_cta = double((ktiles + s - 1) / s) + 2.0;
        const int waves = (ctas + slots - 1) / slots;
        int busiest = (ctas + num_sms - 1) / num_sms;   // CTAs per SM when spread
        if (busiest > ctas_per_sm) busiest = ctas_per_sm;
        const double eff = busiest >= 2 ? 1.0 : 0.6;
        const double t = per_cta * (double)busiest / eff * (double)waves + (s > 1 ? 1.5 : 0.0);
        if (t < best_t - 1e-9) { best_t = t; best = s; }
    }
    return best;
}

}  // namespace dd

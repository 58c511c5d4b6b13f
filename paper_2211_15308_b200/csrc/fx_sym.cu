// Packed-symmetric dense fractional term (3D, SURVEY §8(a) row a-3 "packed-symmetric F (upper
// triangle only) halves the bytes read"; F = (MU)Λ^t(MU)^T is symmetric, Eq.(7)).
//
//   q[:, c] = γ_c F p[:, c] + D[:, c]       (8 columns per grid row y; padded face layout, NP rows)
//
// Storage: F in 128 x 128 blocks (NB = NP/128 block rows), only blocks (I, J) with I <= J in
// row-major block order b(I, J) = I NB - I(I-1)/2 + (J - I); a block is two half-blocks of 64 rows
// x 128 columns, each row-major and contiguous (64 KB), so the packed matrix is one sequential
// stream.  CTA g of a one-per-SM grid takes blocks [g nb/G, (g+1) nb/G) and streams their halves
// through a 3-deep cp.async ring (XOR-swizzled rows: conflict-free fragment loads without
// padding).  Every stored block is used twice, by warps with fixed roles:
//   direct      y_I += F_IJ x_J       warps 0-3: 16 block rows of each half, K = 128 columns;
//               accumulated in registers across the CTA's blocks of one block row
//   transposed  y_J += F_IJ^T x_I     warps 4-7: 32 block columns, K = the half's 64 rows,
//     (I < J)   summed over both halves in registers — no cross-warp reduction
// (x_I, x_J slices staged in smem per block with the ring).
// (32 MMAs per warp per half either way).  Outputs: one direct partial per (block row, CTA
// segment) and one transposed partial per off-diagonal block; k_fx_sym_reduce sums, for block row
// I, the direct segments then T_{J',I} (J' = 0..I-1) in that fixed order and applies the
// epilogue — bitwise reproducible.  Bytes: 8 NP^2/2 (F) + 8 KB per off-diagonal block per 8
// columns (partials, written once, read once) instead of 8 NP^2.
#include <algorithm>
#include <vector>

#include "dd_internal.h"

namespace dd {

namespace {
constexpr int BT = 128, HR = 64, THREADS = 256;
constexpr int BLOCK_ELEMS = BT * BT;          // 16384 doubles
constexpr int XLD = BT + 4;                   // x-slice row stride (conflict-free fragment loads)
// CS (class-sparse, the sine-domain H̃ at N = 128): each 64-row half of a block holds only its one
// nonzero 64-column quadrant — half the bytes and the MMAs; a deeper ring of the 32 KB halves
template <bool CS> struct FxCfg {
    static constexpr int HW = CS ? 64 : BT;             // stored columns per half
    static constexpr int HALF = HR * HW;                 // doubles per half (64 KB / 32 KB)
    static constexpr int STAGES = CS ? 5 : 3;
    // x slices of block b' ride in the cp.async group of its first half (issued STAGES - 1 halves
    // ahead), so up to 1 + STAGES / 2 blocks' slices are live at once
    static constexpr int NXB = 1 + STAGES / 2;
    static constexpr size_t SMEM = ((size_t)STAGES * HALF + (size_t)NXB * 2 * 8 * XLD) * sizeof(double);
};
constexpr size_t SMEM_MAX = FxCfg<false>::SMEM > FxCfg<true>::SMEM ? FxCfg<false>::SMEM : FxCfg<true>::SMEM;

__device__ __forceinline__ void cp16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void mma(double (&c)[4], double a0, double a1, double b) {
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                 : "d"(a0), "d"(a1), "d"(b));
}
// swizzled smem index of half-block element (r, c), rows of HW doubles: the column's bits 2-3 XOR
// the row's bits 0-1
template <int HW>
__device__ __forceinline__ int swz(int r, int c) { return r * HW + (c ^ ((r & 3) << 2)); }
__host__ __device__ __forceinline__ int seg_b0(int g, int nb, int G) { return (int)((long long)g * nb / G); }
}  // namespace

template <bool CS>
__global__ void __launch_bounds__(THREADS, 1)
    k_fx_sym(const double* __restrict__ Fp, const int2* __restrict__ blk, int nblocks, long long NP,
             const double* __restrict__ x, int ncols, double* __restrict__ Dpart, double* __restrict__ Tpart) {
    using C = FxCfg<CS>;
    constexpr int HW = C::HW, HALF = C::HALF, STAGES = C::STAGES, NXB = C::NXB;
    extern __shared__ __align__(16) double sm[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, gq = lane >> 2, tq = lane & 3;
    const int cg = blockIdx.y;                               // group of 8 columns
    const int b0 = seg_b0(blockIdx.x, nblocks, gridDim.x), b1 = seg_b0(blockIdx.x + 1, nblocks, gridDim.x);
    const long long u0 = 2LL * b0, u1 = 2LL * b1;            // half-block units
    const size_t pstride = (size_t)nblocks * BT * 8;          // partial buffers per column group
    double* Dp = Dpart + (size_t)cg * pstride;
    double* Tp = Tpart + (size_t)cg * pstride;
    const bool direct = warp < 4;
    const int w4 = warp & 3;
    const int NB = (int)(NP / BT);

    // x slices of block b: [b % NXB][I | J][n][k] (zero columns past ncols), staged with the ring
    double* xs = sm + (size_t)STAGES * HALF;
    auto load_x = [&](int b) {                               // 2 x 8 x 128 doubles, 4 chunks per thread
        const int2 IJ = blk[b];
#pragma unroll
        for (int j = 0; j < 2 * 8 * BT / 2 / THREADS; j++) {
            const int ch = tid + j * THREADS, which = ch >> 9, n = (ch >> 6) & 7, k2 = (ch & 63) * 2;
            double* dst = xs + (((size_t)(b % NXB) * 2 + which) * 8 + n) * XLD + k2;
            if (cg * 8 + n < ncols)
                cp16(dst, x + (size_t)(cg * 8 + n) * NP + (size_t)(which ? IJ.y : IJ.x) * BT + k2);
            else
                dst[0] = dst[1] = 0.0;
        }
    };
    auto load_half = [&](long long u) {                      // + the block's x slices with its first half
        if ((u & 1) == 0) load_x((int)(u >> 1));
        const double* src = Fp + (size_t)u * HALF;
        double* dst = sm + (size_t)((u - u0) % STAGES) * HALF;
#pragma unroll
        for (int j = 0; j < HALF / 2 / THREADS; j++) {       // 16-byte chunks
            const int ch = tid + j * THREADS;
            const int r = ch / (HW / 2), c2 = (ch % (HW / 2)) * 2;
            cp16(dst + swz<HW>(r, c2), src + (size_t)r * HW + c2);
        }
    };
#pragma unroll
    for (int s = 0; s < STAGES - 1; s++) {
        if (u0 + s < u1) load_half(u0 + s);
        asm volatile("cp.async.commit_group;\n" ::);
    }
    double acc[2][4];                // direct: [half] row-run accumulators; transposed: [output column half] block outputs
#pragma unroll
    for (int h = 0; h < 2; h++) acc[h][0] = acc[h][1] = acc[h][2] = acc[h][3] = 0.0;
    int seg_first = b0;              // first block of the current direct segment
    int2 IJ = b0 < b1 ? blk[b0] : make_int2(0, 0);           // then walked arithmetically (row-major upper blocks)
    int slot = 0;                                            // ring slot of the current half
    double bx[32];                                           // the B fragments of this block (x_J or x_I)
    for (int b = b0; b < b1; b++) {
        const bool offdiag = IJ.x != IJ.y;
        // CS: half h (block rows 64h..) holds the block columns 64 (h ^ cIJ) .. (face row classes of I, J)
        const int cIJ = CS ? (((IJ.x >= NB / 2) ? 1 : 0) ^ ((IJ.y >= NB / 2) ? 1 : 0)) : 0;
        if (!direct) {
#pragma unroll
            for (int m = 0; m < 2; m++) acc[m][0] = acc[m][1] = acc[m][2] = acc[m][3] = 0.0;
        }
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const long long u = 2LL * b + h;
            asm volatile("cp.async.wait_group %0;\n" ::"n"(STAGES - 2));
            __syncthreads();
            if (u + STAGES - 1 < u1) load_half(u + STAGES - 1);
            asm volatile("cp.async.commit_group;\n" ::);
            const double* S = sm + (size_t)slot * HALF;
            slot = slot + 1 == STAGES ? 0 : slot + 1;
            if (h == 0) {                                     // this block's B fragments from the staged slices
                const double* xr = xs + (((size_t)(b % NXB) * 2 + (direct ? 1 : 0)) * 8 + gq) * XLD + tq;
#pragma unroll
                for (int k = 0; k < 32; k++) bx[k] = xr[4 * k];
            }
            const int hp = h ^ cIJ;                           // CS: the stored column half
            if (direct) {
                // rows 16 w4 + gq (+8) of this half, K = its stored columns (block columns 64 hp .. under CS)
                const int r = 16 * w4 + gq;
                if constexpr (CS) {
                    // compile-time register indices on both branches (hp is uniform per block)
                    if (hp == 0) {
#pragma unroll
                        for (int kk = 0; kk < HW; kk += 4)
                            mma(acc[h], S[swz<HW>(r, kk + tq)], S[swz<HW>(r + 8, kk + tq)], bx[kk / 4]);
                    } else {
#pragma unroll
                        for (int kk = 0; kk < HW; kk += 4)
                            mma(acc[h], S[swz<HW>(r, kk + tq)], S[swz<HW>(r + 8, kk + tq)], bx[16 + kk / 4]);
                    }
                } else {
#pragma unroll
                    for (int kk = 0; kk < BT; kk += 4)
                        mma(acc[h], S[swz<HW>(r, kk + tq)], S[swz<HW>(r + 8, kk + tq)], bx[kk / 4]);
                }
            } else if (offdiag) {
                if constexpr (CS) {
                    // outputs: block columns 64 hp + 16 w4 + gq (+8); K = this half's 64 rows
                    const int m = 16 * w4 + gq;
                    if (hp == 0) {
#pragma unroll
                        for (int kk = 0; kk < HR; kk += 4)
                            mma(acc[0], S[swz<HW>(kk + tq, m)], S[swz<HW>(kk + tq, m + 8)], bx[(h * HR + kk) / 4]);
                    } else {
#pragma unroll
                        for (int kk = 0; kk < HR; kk += 4)
                            mma(acc[1], S[swz<HW>(kk + tq, m)], S[swz<HW>(kk + tq, m + 8)], bx[(h * HR + kk) / 4]);
                    }
                } else {
                    // outputs: block columns 32 w4 + 16 mt + gq (+8); K = this half's 64 rows
#pragma unroll
                    for (int mt = 0; mt < 2; mt++) {
                        const int m = 32 * w4 + 16 * mt + gq;
#pragma unroll
                        for (int kk = 0; kk < HR; kk += 4)
                            mma(acc[mt], S[swz<HW>(kk + tq, m)], S[swz<HW>(kk + tq, m + 8)], bx[(h * HR + kk) / 4]);
                    }
                }
            }
        }
        if (direct) {
            // end of this CTA's run of block row I: write the segment's partial (slot = its first block)
            const bool row_end = b + 1 == b1 || IJ.y + 1 == NB;
            if (row_end) {
                double* d = Dp + (size_t)seg_first * BT * 8;
#pragma unroll
                for (int h = 0; h < 2; h++) {
                    const int r = h * HR + 16 * w4 + gq;
                    d[(2 * tq) * BT + r] = acc[h][0];
                    d[(2 * tq + 1) * BT + r] = acc[h][1];
                    d[(2 * tq) * BT + r + 8] = acc[h][2];
                    d[(2 * tq + 1) * BT + r + 8] = acc[h][3];
                    acc[h][0] = acc[h][1] = acc[h][2] = acc[h][3] = 0.0;
                }
                seg_first = b + 1;
            }
        } else if (offdiag) {
            double* t = Tp + (size_t)b * BT * 8;              // Tp[b][n][row of block column J]
#pragma unroll
            for (int mt = 0; mt < 2; mt++) {
                const int m = CS ? 64 * mt + 16 * w4 + gq : 32 * w4 + 16 * mt + gq;
                t[(2 * tq) * BT + m] = acc[mt][0];
                t[(2 * tq + 1) * BT + m] = acc[mt][1];
                t[(2 * tq) * BT + m + 8] = acc[mt][2];
                t[(2 * tq + 1) * BT + m + 8] = acc[mt][3];
            }
        }
        if (++IJ.y == NB) { IJ.x++; IJ.y = IJ.x; }
    }
    asm volatile("cp.async.wait_all;\n" ::);
}

// q[row + c NP] = γ_c (Σ_segments D + Σ_{J'<I} T_{J',I})[row, c] + Dd[row + c NP]
// One CTA per (block row I, column group, half of the 1024 outputs): the contributions of block row I — its direct segment
// partials (CTA order) then T_{0..I-1,I} — are split into RCH chunks summed by RCH thread groups in
// parallel, each in its own fixed order, then the chunk sums in chunk order: a fixed tree,
// bitwise reproducible.
constexpr int RCH = 8, RTH = 64, ROUT = 2;    // chunks x threads per chunk (8 outputs each) x output halves
__global__ void __launch_bounds__(RCH * RTH)
    k_fx_sym_reduce(const double* __restrict__ Dpart, const double* __restrict__ Tpart, int NB, int nblocks, int G,
                    long long NP, int ncols, const int* __restrict__ col_param, int n_param,
                    const double* __restrict__ gp, const double* __restrict__ Dd, double* __restrict__ q) {
    __shared__ double4 part[RCH - 1][RTH][2];
    const int I = blockIdx.x, cg = blockIdx.y;
    const int ch = threadIdx.x / RTH, t = threadIdx.x % RTH;
    const int o0 = (blockIdx.z * RTH + t) * 8; // outputs o0..o0+7 of the 1024 = [n][row] of this block row
    const size_t pstride = (size_t)nblocks * BT * 8;
    const double* Dp = Dpart + (size_t)cg * pstride;
    const double* Tp = Tpart + (size_t)cg * pstride;
    const int rb = (int)((long long)I * NB - (long long)I * (I - 1) / 2), re = rb + (NB - I);
    // the CTAs whose block ranges meet [rb, re): g_first .. g_last
    int g0 = (int)((long long)rb * G / nblocks);
    while (g0 > 0 && seg_b0(g0, nblocks, G) > rb) g0--;
    while (g0 + 1 < G && seg_b0(g0 + 1, nblocks, G) <= rb) g0++;
    int nseg = 0;
    for (int g = g0; g < G && seg_b0(g, nblocks, G) < re; g++) nseg++;
    const int ncon = nseg + I;
    // contribution j: j < nseg -> direct segment of CTA g0 + j;  else T_{j - nseg, I}
    const int per = (ncon + RCH - 1) / RCH, j0 = ch * per, j1 = min(ncon, j0 + per);
    double4 a = make_double4(0, 0, 0, 0), b = make_double4(0, 0, 0, 0);
    for (int j = j0; j < j1; j++) {
        const double* src;
        if (j < nseg) {
            const int slot = max(rb, seg_b0(g0 + j, nblocks, G));
            src = Dp + (size_t)slot * BT * 8;
        } else {
            const int J = j - nseg;
            src = Tp + (size_t)((long long)J * NB - (long long)J * (J - 1) / 2 + (I - J)) * BT * 8;
        }
        const double4 v0 = *reinterpret_cast<const double4*>(src + o0);
        const double4 v1 = *reinterpret_cast<const double4*>(src + o0 + 4);
        a.x += v0.x; a.y += v0.y; a.z += v0.z; a.w += v0.w;
        b.x += v1.x; b.y += v1.y; b.z += v1.z; b.w += v1.w;
    }
    if (ch > 0) { part[ch - 1][t][0] = a; part[ch - 1][t][1] = b; }
    __syncthreads();
    if (ch != 0) return;
#pragma unroll
    for (int k = 0; k < RCH - 1; k++) {
        const double4 u = part[k][t][0], w = part[k][t][1];
        a.x += u.x; a.y += u.y; a.z += u.z; a.w += u.w;
        b.x += w.x; b.y += w.y; b.z += w.z; b.w += w.w;
    }
    const int n = o0 / BT, r0 = o0 % BT;      // 8 outputs share the column n (BT multiple of 8)
    const int colg = cg * 8 + n;
    if (colg >= ncols) return;
    int p = col_param[colg];
    p = p < 0 ? 0 : (p >= n_param ? n_param - 1 : p);
    const double g = gp ? gp[p] : 1.0;
    const size_t o = (size_t)colg * NP + (size_t)I * BT + r0;
    const double y[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    if (Dd) {
#pragma unroll
        for (int k = 0; k < 8; k++) q[o + k] = fma(g, y[k], Dd[o + k]);
    } else {
#pragma unroll
        for (int k = 0; k < 8; k++) q[o + k] = g * y[k];
    }
}

// full row-major NP x NP F -> packed upper blocks, class-sparse: per half h of block (I, J) the 64 x 64
// quadrant at block columns 64 (h ^ c(I) ^ c(J)), c(I) = I >= NB/2 (the face row's parity class)
__global__ void k_fx_pack_cs(const double* __restrict__ F, long long NP, const int2* __restrict__ blk, int nblocks,
                             double* __restrict__ Fp) {
    const int NB = (int)(NP / BT);
    const size_t total = (size_t)nblocks * BLOCK_ELEMS / 2;
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
        const size_t b = idx / (BLOCK_ELEMS / 2), e = idx % (BLOCK_ELEMS / 2);
        const int h = (int)(e / (HR * 64)), r = (int)((e / 64) % HR), k = (int)(e % 64);
        const int2 IJ = blk[b];
        const int hp = h ^ (IJ.x >= NB / 2 ? 1 : 0) ^ (IJ.y >= NB / 2 ? 1 : 0);
        Fp[idx] = F[((size_t)IJ.x * BT + h * HR + r) * NP + (size_t)IJ.y * BT + hp * 64 + k];
    }
}
// full row-major NP x NP F -> packed upper blocks (row-major 128 x 128 each: two 64-row halves)
__global__ void k_fx_pack(const double* __restrict__ F, long long NP, const int2* __restrict__ blk, int nblocks,
                          double* __restrict__ Fp) {
    const size_t total = (size_t)nblocks * BLOCK_ELEMS;
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
        const size_t b = idx / BLOCK_ELEMS, e = idx % BLOCK_ELEMS;
        const int r = (int)(e / BT), k = (int)(e % BT);
        const int2 IJ = blk[b];
        Fp[idx] = F[((size_t)IJ.x * BT + r) * NP + (size_t)IJ.y * BT + k];
    }
}

int fx_sym_blocks(long long NP) {
    const int NB = (int)(NP / BT);
    return NB * (NB + 1) / 2;
}
size_t fx_sym_packed_doubles(long long NP, bool class_sparse) {
    return (size_t)fx_sym_blocks(NP) * BLOCK_ELEMS / (class_sparse ? 2 : 1);
}
size_t fx_sym_partial_doubles(long long NP, int max_cols) {
    return (size_t)fx_sym_blocks(NP) * BT * 8 * (size_t)((max_cols + 7) / 8);
}
bool fx_sym_supported(long long NP) { return NP % BT == 0 && NP >= BT; }

void fx_sym_block_table(long long NP, std::vector<int>& ij) {
    const int NB = (int)(NP / BT);
    ij.clear();
    for (int I = 0; I < NB; I++)
        for (int J = I; J < NB; J++) { ij.push_back(I); ij.push_back(J); }
}

cudaError_t fx_sym_pack(const double* F, long long NP, const int* blk, double* Fp, cudaStream_t st, bool class_sparse) {
    if (class_sparse)
        k_fx_pack_cs<<<148 * 8, 256, 0, st>>>(F, NP, reinterpret_cast<const int2*>(blk), fx_sym_blocks(NP), Fp);
    else
        k_fx_pack<<<148 * 8, 256, 0, st>>>(F, NP, reinterpret_cast<const int2*>(blk), fx_sym_blocks(NP), Fp);
    return cudaGetLastError();
}

cudaError_t fx_sym_apply(const double* Fp, const int* blk, long long NP, const double* p, double* q, const double* D,
                         int ncols, const int* col_param, int n_param, const double* gp, double* Dpart, double* Tpart,
                         int num_sms, cudaStream_t st, bool class_sparse) {
    if (ncols <= 0) return cudaSuccess;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_fx_sym<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)FxCfg<false>::SMEM);
        if (e == cudaSuccess)
            e = cudaFuncSetAttribute(k_fx_sym<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)FxCfg<true>::SMEM);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const int nb = fx_sym_blocks(NP), NB = (int)(NP / BT), ncg = (ncols + 7) / 8;
    const int G = std::min(nb, num_sms);
    if (class_sparse)
        k_fx_sym<true><<<dim3(G, ncg), THREADS, FxCfg<true>::SMEM, st>>>(Fp, reinterpret_cast<const int2*>(blk), nb, NP, p,
                                                                        ncols, Dpart, Tpart);
    else
        k_fx_sym<false><<<dim3(G, ncg), THREADS, FxCfg<false>::SMEM, st>>>(Fp, reinterpret_cast<const int2*>(blk), nb, NP,
                                                                          p, ncols, Dpart, Tpart);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_fx_sym_reduce<<<dim3(NB, ncg, ROUT), RCH * RTH, 0, st>>>(Dpart, Tpart, NB, nb, G, NP, ncols, col_param, n_param, gp, D,
                                                          q);
    return cudaGetLastError();
}

}  // namespace dd

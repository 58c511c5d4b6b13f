// Packed-symmetric dense fractional term (3D, SURVEY §8(a) row a-3 "packed-symmetric F (upper
// triangle only) halves the bytes read"; F = (MU)Λ^t(MU)^T is symmetric, Eq.(7)).
//
//   q[:, c] = γ_c F p[:, c] + D[:, c]       (8 columns per grid row y; padded face layout, NP rows)
//
// Storage: F in 128 x 128 blocks (NB = NP/128 block rows), only blocks (I, J) with I <= J, block
// index b(I, J) = I NB - I(I-1)/2 + (J - I); a block is 8 slabs of 128 rows x 16 columns, each
// slab row-major and contiguous (16 KB), so the whole packed matrix is one sequential stream.
// One pass reads every stored block once and uses it twice:
//   direct      y_I += F_IJ x_J          (all 8 warps, 16 rows each, 4 m16n8k4 DMMA per slab)
//   transposed  y_J += F_IJ^T x_I  (I<J) (every warp its 16 block rows as the K-range, 4 DMMA
//               per slab; the 8 warp partials summed in fixed order once per block)
// Each block's two 128 x 8 contributions go to partial buffers; k_fx_sym_reduce sums, for block
// row I, D_{I,J} (J = I..NB-1) then T_{J',I} (J' = 0..I-1) in that fixed order and applies the
// epilogue — bitwise reproducible.  Bytes: 8 NP^2/2 (F) + 2 x 8 KB per block per 8 columns
// (partials, written once, read once) instead of 8 NP^2.
#include <algorithm>
#include <vector>

#include "dd_internal.h"

namespace dd {

namespace {
constexpr int BT = 128, SLAB = 32, NSLAB = BT / SLAB, LDSL = SLAB + 4, STAGES = 3, THREADS = 256;
constexpr int MT = SLAB / 16;                 // 16-row output tiles of the transposed product per slab
constexpr int SLAB_ELEMS = BT * SLAB;         // 4096 doubles = 32 KB
constexpr int BLOCK_ELEMS = BT * BT;          // 16384 doubles
constexpr int XS = 2 * 8 * BT;                 // one block's x_I and x_J slices: [I|J][col][row]
constexpr int RED = (THREADS / 32) * NSLAB * SLAB * 8;   // per-warp transposed partials of one block
constexpr size_t SMEM = ((size_t)STAGES * BT * LDSL + RED + 2 * XS) * sizeof(double);

__device__ __forceinline__ void cp16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void mma(double (&c)[4], double a0, double a1, double b) {
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
                 : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
                 : "d"(a0), "d"(a1), "d"(b));
}
}  // namespace

__global__ void __launch_bounds__(THREADS, 1)
    k_fx_sym(const double* __restrict__ Fp, const int2* __restrict__ blk, int nblocks, long long NP,
             const double* __restrict__ x, int ncols, double* __restrict__ Dpart, double* __restrict__ Tpart) {
    extern __shared__ __align__(16) double sm[];
    double* red = sm + (size_t)STAGES * BT * LDSL;          // [warp][slab][n][m]: transposed partials
    double* xs = red + RED;                                  // [block parity][I|J][col][row], cp.async-staged
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, gq = lane >> 2, tq = lane & 3;
    const int cg = blockIdx.y;                               // group of 8 columns
    const int b0 = (int)((long long)blockIdx.x * nblocks / gridDim.x);
    const int b1 = (int)((long long)(blockIdx.x + 1) * nblocks / gridDim.x);
    const long long u0 = (long long)b0 * NSLAB, u1 = (long long)b1 * NSLAB;
    const int col = cg * 8 + gq;                             // this lane's B-fragment column
    const bool colok = col < ncols;
    const double* xc = x + (size_t)(colok ? col : 0) * NP;
    const size_t pstride = (size_t)nblocks * BT * 8;          // partial buffers per column group
    double* Dp = Dpart + (size_t)cg * pstride;
    double* Tp = Tpart + (size_t)cg * pstride;

    auto load_slab = [&](long long u) {
        const double* src = Fp + (size_t)u * SLAB_ELEMS;
        double* dst = sm + (size_t)((u - u0) % STAGES) * BT * LDSL;
#pragma unroll
        for (int j = 0; j < SLAB_ELEMS / 2 / THREADS; j++) {   // 16-byte chunks
            const int ch = tid + j * THREADS;
            const int r = ch / (SLAB / 2), k2 = (ch % (SLAB / 2)) * 2;
            cp16(dst + r * LDSL + k2, src + (size_t)r * SLAB + k2);
        }
    };
    // x slices of block b (rows of block row I and block column J, 8 columns) -> xs[b & 1], issued
    // one block ahead inside the slab ring's commit groups (ready when the block's first slab is)
    auto load_x = [&](int b) {
        const int2 IJ = blk[b];
        double* dst = xs + (size_t)(b & 1) * XS;
#pragma unroll
        for (int j = 0; j < XS / 2 / THREADS; j++) {            // 16-byte chunks: 4 per thread
            const int ch = tid + j * THREADS;
            const int which = ch >> 9, c = (ch >> 6) & 7, r2 = (ch & 63) * 2;
            const int cc = cg * 8 + c < ncols ? cg * 8 + c : 0;
            const size_t row = (size_t)(which ? IJ.y : IJ.x) * BT + r2;
            cp16(dst + which * 8 * BT + c * BT + r2, x + (size_t)cc * NP + row);
        }
    };
#pragma unroll
    for (int s = 0; s < STAGES - 1; s++) {
        if (u0 + s < u1) load_slab(u0 + s);
        if (s == 0 && b0 < b1) load_x(b0);
        asm volatile("cp.async.commit_group;\n" ::);
    }
    for (int b = b0; b < b1; b++) {
        const int2 IJ = blk[b];
        const bool offdiag = IJ.x != IJ.y;
        double bI[4], bJ[NSLAB][SLAB / 4];
        double* xb = xs + (size_t)(b & 1) * XS;
        double accD[4] = {0.0, 0.0, 0.0, 0.0};
        double accT[NSLAB][MT][4];
#pragma unroll
        for (int s = 0; s < NSLAB; s++) {
            const long long u = (long long)b * NSLAB + s;
            asm volatile("cp.async.wait_group %0;\n" ::"n"(STAGES - 2));
            __syncthreads();
            if (u + STAGES - 1 < u1) load_slab(u + STAGES - 1);
            if (s == 0 && b + 1 < b1) load_x(b + 1);      // completes with slab u + 5 <= next block's slab 0
            asm volatile("cp.async.commit_group;\n" ::);
            if (s == 0) {
                // this block's x fragments from the staged slices (zero for columns >= ncols)
#pragma unroll
                for (int j = 0; j < 4; j++) bI[j] = colok ? xb[gq * BT + warp * 16 + 4 * j + tq] : 0.0;
#pragma unroll
                for (int s2 = 0; s2 < NSLAB; s2++)
#pragma unroll
                    for (int j = 0; j < SLAB / 4; j++)
                        bJ[s2][j] = colok ? xb[8 * BT + gq * BT + s2 * SLAB + 4 * j + tq] : 0.0;
            }
            const double* S = sm + (size_t)((u - u0) % STAGES) * BT * LDSL;
            // direct: rows 16 warp .. +16 of the block, K = this slab's 16 columns (block column J)
            const double* a = S + (warp * 16 + gq) * LDSL + tq;
#pragma unroll
            for (int kk = 0; kk < SLAB; kk += 4) mma(accD, a[kk], a[8 * LDSL + kk], bJ[s][kk / 4]);
            // transposed: outputs = the slab's 16 columns (rows J*128 + 16 s + m of y), K = this warp's
            // 16 block rows (At[m][k] = S[16 warp + k][m]); partial over the warp's K-range
#pragma unroll
            for (int mt = 0; mt < MT; mt++) {
                accT[s][mt][0] = accT[s][mt][1] = accT[s][mt][2] = accT[s][mt][3] = 0.0;
                if (offdiag) {
                    const double* at = S + (warp * 16 + tq) * LDSL + mt * 16 + gq;
#pragma unroll
                    for (int j = 0; j < 4; j++) mma(accT[s][mt], at[4 * j * LDSL], at[4 * j * LDSL + 8], bI[j]);
                }
            }
        }
        // direct partial of block (I, J): rows (16 warp + gq | + 8), columns (2 tq | 2 tq + 1)
        {
            double* d = Dp + (size_t)b * BT * 8;
            const int r = warp * 16 + gq;
            d[(2 * tq) * BT + r] = accD[0];
            d[(2 * tq + 1) * BT + r] = accD[1];
            d[(2 * tq) * BT + r + 8] = accD[2];
            d[(2 * tq + 1) * BT + r + 8] = accD[3];
        }
        if (offdiag) {
            // sum the 8 warps' K-range partials in fixed warp order
            // red[warp][n][row of the block's column range] (8 x 128 per warp)
#pragma unroll
            for (int s = 0; s < NSLAB; s++)
#pragma unroll
                for (int mt = 0; mt < MT; mt++) {
                    double* rw = red + (size_t)warp * 8 * BT + s * SLAB + mt * 16;
                    rw[(2 * tq) * BT + gq] = accT[s][mt][0];
                    rw[(2 * tq + 1) * BT + gq] = accT[s][mt][1];
                    rw[(2 * tq) * BT + gq + 8] = accT[s][mt][2];
                    rw[(2 * tq + 1) * BT + gq + 8] = accT[s][mt][3];
                }
            __syncthreads();
            double* t = Tp + (size_t)b * BT * 8;
#pragma unroll
            for (int j = 0; j < 8 * BT / THREADS; j++) {
                const int o = tid + j * THREADS;           // output index n * 128 + row
                double v = 0.0;
#pragma unroll
                for (int w = 0; w < THREADS / 32; w++) v += red[(size_t)w * 8 * BT + o];
                t[o] = v;                                  // Tp[b][n][row]
            }
        }
    }
    asm volatile("cp.async.wait_all;\n" ::);
}

// q[row + c NP] = γ_c (Σ_{J>=I} D_{I,J} + Σ_{J'<I} T_{J',I})[row, c] + Dd[row + c NP]
// One CTA per (block row I, column group): RCH chunks of the NB contributions (D_{I,I..NB-1} then
// T_{0..I-1,I}, in that order) are summed by RCH thread groups in parallel, each in its own fixed
// order, then the chunk sums in chunk order — a fixed tree, bitwise reproducible.
constexpr int RCH = 4, RTH = 128;             // chunks x threads per chunk; 8 outputs per thread
__global__ void __launch_bounds__(RCH * RTH)
    k_fx_sym_reduce(const double* __restrict__ Dpart, const double* __restrict__ Tpart, int NB, int nblocks,
                    long long NP, int ncols, const int* __restrict__ col_param, int n_param,
                    const double* __restrict__ gp, const double* __restrict__ Dd, double* __restrict__ q) {
    __shared__ double4 part[RCH - 1][RTH][2];
    const int I = blockIdx.x, cg = blockIdx.y;
    const int ch = threadIdx.x / RTH, t = threadIdx.x % RTH;
    const int o0 = t * 8;                     // outputs o0..o0+7 of the 1024 = [n][row] of this block row
    const size_t pstride = (size_t)nblocks * BT * 8;
    const double* Dp = Dpart + (size_t)cg * pstride;
    const double* Tp = Tpart + (size_t)cg * pstride;
    const long long rowbase = (long long)I * NB - (long long)I * (I - 1) / 2;
    // contribution j in [0, NB): j < NB - I -> D_{I, I + j};  else T_{j - (NB - I), I}
    const int per = (NB + RCH - 1) / RCH, j0 = ch * per, j1 = min(NB, j0 + per);
    double4 a = make_double4(0, 0, 0, 0), b = make_double4(0, 0, 0, 0);
#pragma unroll 4
    for (int j = j0; j < j1; j++) {
        const double* src;
        if (j < NB - I) {
            src = Dp + (size_t)(rowbase + j) * BT * 8;
        } else {
            const int J = j - (NB - I);
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
    const double g = gp[p];
    const size_t o = (size_t)colg * NP + (size_t)I * BT + r0;
    const double y[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
    for (int k = 0; k < 8; k++) q[o + k] = fma(g, y[k], Dd[o + k]);
}

// full row-major NP x NP F -> packed upper blocks
__global__ void k_fx_pack(const double* __restrict__ F, long long NP, const int2* __restrict__ blk, int nblocks,
                          double* __restrict__ Fp) {
    const size_t total = (size_t)nblocks * BLOCK_ELEMS;
    for (size_t idx = blockIdx.x * (size_t)blockDim.x + threadIdx.x; idx < total; idx += (size_t)gridDim.x * blockDim.x) {
        const size_t b = idx / BLOCK_ELEMS, e = idx % BLOCK_ELEMS;
        const int s = (int)(e / SLAB_ELEMS), r = (int)((e % SLAB_ELEMS) / SLAB), k = (int)(e % SLAB);
        const int2 IJ = blk[b];
        Fp[idx] = F[((size_t)IJ.x * BT + r) * NP + (size_t)IJ.y * BT + s * SLAB + k];
    }
}

int fx_sym_blocks(long long NP) {
    const int NB = (int)(NP / BT);
    return NB * (NB + 1) / 2;
}
size_t fx_sym_packed_doubles(long long NP) { return (size_t)fx_sym_blocks(NP) * BLOCK_ELEMS; }
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

cudaError_t fx_sym_pack(const double* F, long long NP, const int* blk, double* Fp, cudaStream_t st) {
    k_fx_pack<<<148 * 8, 256, 0, st>>>(F, NP, reinterpret_cast<const int2*>(blk), fx_sym_blocks(NP), Fp);
    return cudaGetLastError();
}

cudaError_t fx_sym_apply(const double* Fp, const int* blk, long long NP, const double* p, double* q, const double* D,
                         int ncols, const int* col_param, int n_param, const double* gp, double* Dpart, double* Tpart,
                         int num_sms, cudaStream_t st) {
    if (ncols <= 0) return cudaSuccess;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(k_fx_sym, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    const int nb = fx_sym_blocks(NP), NB = (int)(NP / BT), ncg = (ncols + 7) / 8;
    const int G = std::min(nb, num_sms);
    k_fx_sym<<<dim3(G, ncg), THREADS, SMEM, st>>>(Fp, reinterpret_cast<const int2*>(blk), nb, NP, p, ncols, Dpart, Tpart);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    k_fx_sym_reduce<<<dim3(NB, ncg), RCH * RTH, 0, st>>>(Dpart, Tpart, NB, nb, NP, ncols, col_param, n_param, gp, D, q);
    return cudaGetLastError();
}

}  // namespace dd

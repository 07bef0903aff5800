// device.hpp -- device-side data structures and kernel launchers shared by the .cu files.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "layout.hpp"

namespace pmfgpu {

// Device copy of one sweep layout (layout.hpp SweepLayout).
struct DevSweep {
    int32_t n_out = 0, gat_extent = 0, panel_size = 0, n_panels = 0, sentinel = 0;
    bool smem = true, idx16 = true;
    int64_t n_entries = 0;
    int32_t n_units = 0, n_mo = 0, ctas = 0, n_slots = 0;
    void* idx = nullptr;          // uint16_t* or int32_t*
    float* R = nullptr;           // residual values (padded layout)
    Unit* units = nullptr;
    int32_t* unit_panel = nullptr;
    Piece* pieces = nullptr;
    int32_t* piece_start = nullptr;
    int32_t* panel_base = nullptr;
    int32_t* mo_out = nullptr;
    int32_t* mo_start = nullptr;
    float2* partial = nullptr;
    int32_t n_mo_big = 0;
    int64_t n_dense = 0;            // partial[p * n_out + o]: first chunk of segment (p, o)
    int32_t n_pieces = 0;
    double avg_segment = 0.0;
    int* gcnt = nullptr;            // 4 per piece (class / chunk counters) + 1 (CTAs done): work stealing
    bool flat = false;              // segmented-stream layout (flat_kernels.cu)
    FlatChunk* chunks = nullptr;
    int32_t* uinfo = nullptr;       // flat: per unit partial slot, or -(output + 1) (direct write)
    int32_t* uout = nullptr;        // flat: per unit output
    uint32_t* tailbits = nullptr;
    bool promote_fused = true;      // else: rmw_sub residual sub-passes + a plain sweep
    int32_t rmw_sub = 1, sub_width = 0;
    uint16_t* usplit = nullptr;     // rmw_sub > 1: per unit rmw_sub+1 offsets
};

// kRmw: the promote's residual update alone (R <- (R - u'v') + [w != 0] w h), no accumulation
enum SweepMode { kPlain = 0, kPromote = 1, kDemote = 2, kRmw = 3 };

// Operands of one sweep.  "g*" vectors are indexed by the gather index (padded space),
// "o*" vectors by the output index (out_off + local output).
struct SweepOperands {
    const float* gn = nullptr;  // num/den vector (v on the CSR side, u on the CSC side)
    const float* ga = nullptr;  // demote factor, gathered   (v' on CSR, u' on CSC)
    const float* gb = nullptr;  // promote factor, gathered  (h  on CSR, w  on CSC)
    const float* oa = nullptr;  // demote factor, per output (u' on CSR, v' on CSC)
    const float* ob = nullptr;  // promote factor, per output(w  on CSR, h  on CSC)
    float* out = nullptr;       // result vector (u or v), written at out_off + o
    int32_t out_off = 0;
    unsigned long long* cta_clock = nullptr;  // profiling: per-CTA [start, end] globaltimer (ns)
    float lambda = 0.f;
    int32_t psz = 0;  // set by the launcher: staged panel width (= the sentinel index of padding entries)
};

// Launches one CCD++ sweep over a layout (ccd.hpp:153-197 with the promote of ccd.hpp:133-151
// and the deferred writeback of ccd.hpp:199-218 fused in when mode == kPromote; kDemote only
// applies R -= oa*ga).  csr_side selects which operand is "w" (the skip test of ccd.hpp:142).
// Also launches the fixed-order finalize for outputs with several units.  Returns the number of
// kernels launched.
int launch_sweep(const DevSweep& L, SweepMode mode, bool csr_side, const SweepOperands& op,
                 cudaStream_t stream);
size_t sweep_smem_bytes(const DevSweep& L, SweepMode mode, bool csr_side);
// Fixed-order finalize of outputs with partial slots (after a sweep).  Returns kernels launched.
int launch_finalize(const DevSweep& L, const SweepOperands& op, cudaStream_t stream);
// Flat layouts: the same contract as launch_sweep, with the segmented-stream kernels.
int launch_flat(const DevSweep& L, SweepMode mode, bool csr_side, const SweepOperands& op, cudaStream_t stream);
void flat_set_attributes(size_t max_smem);
// A whole CCD++ outer iteration for small single-panel layouts in one cluster kernel (small_kernels.cu).
// Eligible: single-panel 16-bit layouts without partial slots whose per-CTA residual runs and the factor
// columns fit one CTA's shared memory (MovieLens-100K: 86 KB).
bool small_ccdpp_eligible(const DevSweep& csr, const DevSweep& csc, const SweepLayout& hcsr, const SweepLayout& hcsc,
                          int32_t m, int32_t n);
cudaError_t launch_small_ccdpp(const DevSweep& csr, const DevSweep& csc, const SweepLayout& hcsr,
                               const SweepLayout& hcsc, float* W, float* H, float* ub, float* vb, int64_t ldm,
                               int64_t ldn, int32_t m, int32_t n, int k, int inner, float lambda, cudaStream_t s);
void sweep_set_attributes(size_t max_smem);

// dst[i * k + t] = src[t * ld + i] for i < count (column-major k x ld factor -> row-major).
void launch_transpose(const float* src, int64_t ld, int k, int32_t count, float* dst, cudaStream_t stream);

// ---- evaluation (model.hpp:103-167) -----------------------------------------------------------
// Factor element (i, t) lives at F[i * si + t * st].
struct FactorView {
    const float* p;
    int64_t si, st;
};

// Per-unit squared-error sums of the CSR layout `L` (values A) into unit_loss[n_units].
void launch_unit_loss(const DevSweep& L, const float* A, int32_t row_off, FactorView W,
                      FactorView H, int k, double* unit_loss, cudaStream_t stream);
// sum of squares of x[0..n) (double) into *out via a fixed-shape reduction (scratch >= 1024).
void launch_sumsq(const float* x, int64_t n, double* scratch, double* out, cudaStream_t stream);
// deterministic sum of x[0..n) into *out.
void launch_sum(const double* x, int64_t n, double* scratch, double* out, cudaStream_t stream);
struct DevTriplet {
    int32_t user, item;
    float rating;
};
// RatingsMatrix::from_triplets (sparse.hpp:73-149) on the device (ingest.cu): CSR + CSC of nnz
// device triplets into device arrays; *bad = first invalid triplet index or -1, *dup = CSR position of
// the first duplicate or -1 (outputs valid only when both are -1).  nnz < 2^31.
size_t ingest_scratch_bytes(int64_t nnz);
cudaError_t ingest_build(const DevTriplet* t, int64_t nnz, int32_t m, int32_t n, void* scratch, int64_t* row_start,
                         int32_t* col_of, float* val_row, int64_t* col_start, int32_t* row_of, float* val_col,
                         int64_t* bad, int64_t* dup, cudaStream_t s);
// sum over probe of (r - predict)^2, predict in FP32 sequential t (model.hpp:103-114).
void launch_probe_sse(const DevTriplet* probe, int64_t n, FactorView W, FactorView H, int k,
                      double* scratch, double* out, cudaStream_t stream);

// ---- item/user-wise CCD (ccd.hpp:52-125), ccdw_kernels.cu -------------------------------------
struct CcdWs {
    int32_t m = 0, n = 0;
    int64_t nnz = 0;
    const int64_t* row_start = nullptr;
    const int32_t* col_of = nullptr;
    const int64_t* col_start = nullptr;
    const int32_t* row_of = nullptr;
    float* R_row = nullptr;      // residual, CSR order
    float* R_col = nullptr;      // residual, CSC order
    int32_t* csr2csc = nullptr;  // position maps (the reference's xlinks)
    int32_t* csc2csr = nullptr;
    float* WT = nullptr;           // k x m column-major copy of W for the H sweep (coalesced gathers)
    int32_t* col_order = nullptr;  // columns longest first (the H sweep claims them in this order)
    int* counter = nullptr;
};
void launch_ccd_xlinks(const int64_t* row_start, const int32_t* col_of, const int64_t* col_start,
                       const int32_t* row_of, int32_t m, int32_t* csr2csc, int32_t* csc2csr, cudaStream_t s);
// One epoch (W sweep, mirror, H sweep, mirror) on row-major W (m x k) / H (n x k).  Returns launches.
int launch_ccd_epoch(const CcdWs& ws, float* W, float* H, int k, float lambda, cudaStream_t s);
// R_row = A - W H^T (t ascending, products rounded before the subtracts), mirrored into R_col.
void launch_ccd_residual(const CcdWs& ws, const float* A_row, const float* W, const float* H, int k, cudaStream_t s);

// ---- top_n (model.hpp:172-209), topn_kernels.cu ------------------------------------------------
// For each of n_users users (W rows users[u]): the `count` best unrated items of W H^T (row-major
// m x k, n x k), excluding ex_items[ex_start[u] .. ex_start[u+1]) (ascending).  out_* are
// n_users x count (items -1 past out_count[u]).
size_t topn_smem_bytes(int k, int count);
void topn_set_attributes(size_t max_smem);
// Any count / k: batches of `batch` users, full scoring + stable segmented radix sort (scratch from
// topn_wide_scratch_bytes).
int topn_wide_batch(int32_t n);
size_t topn_wide_scratch_bytes(int32_t n, int batch);
cudaError_t launch_topn_wide(const float* W, const float* H, int32_t n, int k, const int32_t* users, int32_t n_users,
                             const int64_t* ex_start, const int32_t* ex_items, int count, int32_t* out_items,
                             float* out_scores, int32_t* out_count, void* scratch, int batch, cudaStream_t s);
void launch_topn(const float* W, const float* H, int32_t n, int k, const int32_t* users, int32_t n_users,
                 const int64_t* ex_start, const int32_t* ex_items, int count, int32_t* out_items, float* out_scores,
                 int32_t* out_count, cudaStream_t s);

// ---- ALS (als.hpp:47-68, dense.hpp:35-124) ------------------------------------------------------
struct DevAls {
    int32_t n_out = 0, n_units = 0, n_mo = 0, n_slots = 0, n_empty = 0;
    int64_t n_entries = 0;
    int32_t* idx = nullptr;
    float* val = nullptr;
    Unit* units = nullptr;
    int32_t* mo_out = nullptr;
    int32_t* mo_start = nullptr;
    int32_t* empty_out = nullptr;
    float* partial = nullptr;   // n_slots * (k*k + k + 1)
    float* big_scratch = nullptr;  // k > 64 with the system past shared memory: per-CTA k x k in HBM
};

// Solves every output row of one side: out row (out_off + o) of the row-major factor `out`
// (stride k) from the row-major opposing factor `opp` (n_opp addressable rows).  status: device int
// set to 4 on a non-positive pivot.  Returns kernels launched.
// gs: item/user-wise CCD instead of ALS -- one Gauss-Seidel sweep on (G + lambda I) x = b starting
// from the current rows of `out` (needs als_gram_gs_supported(k); returns -1 otherwise).
int launch_als_half(const DevAls& L, const float* opp, int64_t n_opp, float* out, int32_t out_off, int k,
                    float lambda, bool weighted, int* d_counter, int* d_status, int sm_count,
                    cudaStream_t stream, bool gs = false);
bool als_gram_gs_supported(int k);
// k <= 48 (als_umma_kernels.cu): the gram on tcgen05 tensor cores (TMEM accumulators), warp-specialised
// persistent CTAs.  The caller resets *d_counter.  Returns false when k is out of range.
bool als_umma_supported(int k);
bool launch_als_umma(const DevAls& L, const float* opp, int64_t n_opp, float* out, int32_t out_off, int k,
                     float lambda, bool weighted, int* d_counter, int* d_status, int sm_count, cudaStream_t s,
                     bool gs);
void als_umma_set_attributes();
// k > 64 (als_big_kernels.cu): a CTA per unit, the system in shared memory (HBM scratch of
// als_big_scratch_floats past ~216).
int64_t als_big_scratch_floats(int k, int sm_count);
int launch_als_big(const DevAls& L, const float* opp, float* out, int32_t out_off, int k, float lambda, bool weighted,
                   int* d_counter, int* d_status, int sm_count, float* gscratch, cudaStream_t s);
void launch_cholesky_big(float* a, float* x, int batch, int k, int* d_status, int sm_count, float* gscratch,
                         cudaStream_t s);
void als_set_attributes();
// Device-built sweep layouts (layout_device.cu): per-(panel, output) segment lengths of a device CSR /
// CSC, the padded residual / index streams filled from it (delta: per segment, padded minus source
// position; layout.hpp SweepLayout::seg_delta), and the rmw sub-panel split points of every unit.
void seg_count_device(const int64_t* start, const int32_t* idx, int32_t n_out, int32_t pg, int32_t np,
                      int32_t* seg_len, cudaStream_t s);
void layout_fill_device(const int64_t* start, const int32_t* idx, const float* val, int32_t n_out, int64_t nnz,
                        int32_t pg, int32_t np, const int64_t* delta, bool idx16, int32_t sentinel, int64_t n_entries,
                        void* out_idx, float* out_val, cudaStream_t s);
void usplit_device(const Unit* units, const int32_t* real, int64_t nu, const uint16_t* idx, int S, int32_t sub_width,
                   uint16_t* out, cudaStream_t s);

// Batched Cholesky factor + solve of `batch` k*k row-major systems in place.
void launch_cholesky_batched(float* a, float* x, int batch, int k, int* d_status,
                             cudaStream_t stream);

}  // namespace pmfgpu

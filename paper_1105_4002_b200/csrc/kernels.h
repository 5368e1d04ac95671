// Internal kernel launchers of libtvreg (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace tvr {

struct SpmvArgs {
  const int64_t* rp;
  const int32_t* col;
  const uint16_t* col16;  // 16-bit window offsets (SpmvVariant::idx16)
  const float* val;
  const float* src;  // gather vector (x for A, r for A^T), local indices
  const float* b;    // non-null: out = A src - b and sum of squares
  float* out;
  float* out_lo;     // non-null (with b): fp32 remainder r - fl32(r)
  const int64_t* item_row;   // nitems+1 row boundaries
  const int32_t* item_slice; // per item slice id (staged)
  const int64_t* slice_item_end;  // per slice: one past its last item (16-bit kernel)
  int64_t nitems;
  const int64_t* win_lo;     // per slice: first gather index of the slice window
  const int32_t* win_len;    // per slice: window length
  int32_t parts, part_len;   // window parts (16-bit kernel): parts * part_len >= window length
  int64_t nrows;
  const uint16_t* part_off;  // (parts-1) x nrows row-relative starts of parts 1..parts-1
  double* part_acc;          // nrows fp64 partial row sums between parts
  double* partials;
  unsigned* counter;
  double* scal;  // non-null: write 1/2-less sum r^2 to scal[0]
  // fused reduce-scatter (VIEWS mode A^T pass, spmv32p_kernel): row i of the output goes to
  // out_peer[o][i] for the owner o of i (out_bounds[o] <= i < out_bounds[o+1]); out_peer[o] is
  // the owner's inbox slot of this rank, offset so that it is indexed by the global row
  float* const* out_peer;
  const int64_t* out_bounds;
  int n_out;
};

struct SpmvVariant {
  int lpr = 8;       // lanes per row
  bool staged = false;
  int unroll = 2;    // 16-byte chunks in flight per lane
  int minb = 1;      // __launch_bounds__ min blocks per SM
  bool idx16 = false;  // 16-bit column offsets inside the staged slice window (6 B per entry)
  bool parts = false;  // (idx16, staged) window cut into parts: spmv16_parts_kernel
  bool half = false;   // padded 16-bit kernel with the window's first part_len entries staged
};
cudaError_t launch_compress_cols(const SpmvArgs& a, const int32_t* col, uint16_t* col16, bool expand,
                                 int32_t* col_out, cudaStream_t st);
cudaError_t launch_parts_rows(const SpmvArgs& a, bool expand, const int32_t* col, uint16_t* col16,
                              uint16_t* part_off, int32_t* col_out, cudaStream_t st);
bool spmv_variant_exists(const SpmvVariant& v);
cudaError_t ensure_smem_attr(const void* func, size_t smem);
cudaError_t launch_spmv(const SpmvArgs& a, const SpmvVariant& v, int grid, int block, size_t smem,
                        cudaStream_t st);
// padded-row 16-bit kernel (rows start on 8-entry boundaries, zero-padded)
cudaError_t launch_spmv16p(const SpmvArgs& a, const SpmvVariant& v, int grid, int block,
                           size_t smem, cudaStream_t st);
int spmv16p_occupancy(const SpmvVariant& v, int block, size_t smem);
// padded-row int32 kernel (global columns; rows on 4-entry boundaries, zero-padded)
cudaError_t launch_spmv32p(const SpmvArgs& a, const SpmvVariant& v, int grid, int block,
                           cudaStream_t st);
int spmv32p_occupancy(const SpmvVariant& v, int block);
cudaError_t launch_inbox_sum(int64_t n, const float* inbox, int64_t stride, int world, float* out,
                             cudaStream_t st);
cudaError_t launch_pad_rows32(int64_t m, const int64_t* rp, const int64_t* rpp, const int32_t* col,
                              const float* val, int32_t* colp, float* valp, cudaStream_t st);
cudaError_t launch_pad_rows(int64_t m, const int64_t* rp, const int64_t* rpp, const uint16_t* col16,
                            const float* val, uint16_t* col16p, float* valp, cudaStream_t st);
int spmv_occupancy(const SpmvVariant& v, int block, size_t smem);

// Sliced-ELL SpMV over 16-bit window offsets (spmv.cu spmv16s_kernel): blocks of 32 rows sorted
// by length inside a slice, chunk-interleaved, one row per lane.
struct SellArgs {
  const int64_t* blk_off;   // per block: first chunk step (a step = 32 lanes x 8 entries)
  const int32_t* blk_k;     // per block: chunk steps (its longest row's chunks)
                            // (per-block arrays are indexed by stored block k % nb)
  const int32_t* blk_slice; // per block: slice (window)
  const int64_t* zend;      // per slice: one past its last block
  const int64_t* cum;       // nblk+1 prefix of per-block work (steps + 2)
  const int32_t* perm;      // 32 per block: row of each lane, -1 for an empty lane
  double* blk_sq;           // per virtual block: sum of its rows' r^2 (scratch, when scal)
  float* const* out_peer;   // spmv32s_kernel, VIEWS A^T: per owner rank, its inbox (row-indexed)
  const int64_t* out_bounds;
  int n_out;
  const double* acc_in;     // column parts after the first: each row starts from acc_in[row]
  double* acc_out;          // column parts before the last: the row's fp64 sum goes here
  const uint16_t* col16;    // [step][lane][8] window offsets (zero pads)
  const int32_t* col32;     // spmv32s_kernel: int32 global columns in 4-entry chunks
  const int64_t* row_start; // spmv32s_kernel row-mode blocks: per slot, row start (chunks)
  const int64_t* rp;        // spmv32s_kernel row-mode blocks: the CSR row pointer (lengths)
  const float* val;         // [step][lane][8] values (zero pads)
  const float* src;
  const float* src_lo;      // non-null: A (src + src_lo) (extended-precision solver iterates,
                            // DESIGN §5.3), the lo parts gathered from global memory, or staged
  int32_t lo_off;           // > 0: after the hi window, lo_off floats on (spmv16s_kernel)
  const float* b;           // non-null: out = A src - b, sum r^2
  float* out;
  float* out_lo;
  int64_t blk_lo, blk_hi;   // virtual blocks [blk_lo, blk_hi): block k % nb of repetition k / nb
  int64_t nb;               // stored blocks
  int32_t rep;              // repetitions (slice-shared operator: slices; else 1)
  int64_t rep_rows;         // output row offset per repetition
  int64_t rep_win;          // gather-window offset per repetition
  int64_t rep_total;        // slice groups (spmv16z_kernel): slices in all groups
  int32_t wstride;          // slice groups: shared-memory floats between staged windows
  const int64_t* win_lo;
  const int32_t* win_len;
  int part_len;             // half: window entries staged
  int32_t l2hint;           // spmv32s_kernel L2 policies: bit 0 matrix stream evict-first,
                            // bit 1 gathered vector evict-last
  int32_t ilv;              // spmv32s_kernel: > 0 = CTA c walks the block chunks c, c + G,
                            // c + 2G, ... of ilv blocks each (the grid sweeps the block order
                            // together: z-ordered blocks keep the gathered sub-volume in L2);
                            // 0 = one contiguous work-balanced range per CTA
  long long* cta_prof;      // diagnostic (TVR_SELL_PROF=1): per CTA start ns, end ns, SM id
  const int64_t* cta_tab;   // non-null: the CTA ranges of a full-range launch with cta_tab_grid
  int32_t cta_tab_grid;     // CTAs, precomputed at plan time (sell_cta_range's search results)
  double* partials;
  unsigned* counter;
  double* scal;
};
// tab[i], i = 0..grid: first virtual block of CTA i of a `grid`-CTA launch over [a.blk_lo,
// a.blk_hi) (tab[grid] = a.blk_hi): exactly what the kernels' own range search returns
cudaError_t launch_sell_cta_table(const SellArgs& a, int grid, int64_t* tab, cudaStream_t st);
struct SellVariant {
  bool staged = true;
  bool half = false;
  bool dyn = true;    // warps take blocks from a shared counter (else round-robin)
  int zgroup = 1;     // slice-shared operator: slices per pass (spmv16z_kernel when > 1)
  int unroll = 2;     // steps of loads in flight per lane
  int block = 512;
};
cudaError_t launch_spmv16s(const SellArgs& a, const SellVariant& v, int grid, size_t smem,
                           cudaStream_t st);
int spmv16s_occupancy(const SellVariant& v, size_t smem);
bool spmv16s_lo_ok(const SellVariant& v);  // an extended-precision (src_lo) instantiation exists
cudaError_t launch_sell_fill(int64_t nslots, const int32_t* perm, const int64_t* blk_off,
                             const int64_t* rp, const int32_t* lo_off, const int32_t* hi_off,
                             uint16_t coff, const uint16_t* col16, const float* val,
                             uint16_t* col16s, float* vals, cudaStream_t st);
cudaError_t launch_spmv32s(const SellArgs& a, int unroll, int grid, cudaStream_t st, int block = 512);
int spmv32s_occupancy(int unroll, int block = 512);
cudaError_t launch_sell_fill32(int64_t nslots, const int32_t* perm, const int64_t* blk_off,
                               const int32_t* blk_k, const int64_t* row_start, const int64_t* rp,
                               const int32_t* col, const float* val, int32_t* cols, float* vals,
                               cudaStream_t st);
// gather layouts of the non-separable A pass (spmv.cu): xs = [x | x_yx | x_bricks] (3N floats);
// per-row mapped and sorted columns; per-block distinct-line counts; the layout-aware fill
cudaError_t launch_relayout(const float* x, float* xs, int nx, int ny, int64_t N, cudaStream_t st);
cudaError_t launch_layout_sort_rows(int64_t rows, const int64_t* rp, const int32_t* col, int L, int nx,
                                    int ny, int64_t N, int32_t* scol, uint8_t* bad, cudaStream_t st);
cudaError_t launch_layout_count(int64_t nblk, int64_t rows, const int64_t* rp, const int32_t* scol,
                                int64_t* cnt_lane, int64_t* cnt_row, cudaStream_t st);
cudaError_t launch_sell_fill32_layout(int64_t nslots, const int32_t* perm, const int64_t* blk_off,
                                      const int32_t* blk_k, const int64_t* row_start,
                                      const uint8_t* layout, const int64_t* rp, const int32_t* col,
                                      const float* val, int nx, int ny, int64_t N, int32_t* cols,
                                      float* vals, cudaStream_t st);
cudaError_t launch_sell32_mode(int64_t nblk, int64_t rows, const int64_t* rp, const int32_t* col,
                               uint8_t* mode, cudaStream_t st, int bias_pct = 100);
// per block of 32 consecutive rows: the z (column / plane) of the middle entry of its middle
// nonempty row, -1 for an empty block (the key of the z-ordered block layout)
cudaError_t launch_sell32_zkey(int64_t nblk, int64_t rows, const int64_t* rp, const int32_t* col,
                               int64_t plane, int32_t* key, cudaStream_t st);
// per row: the first entry offset (from rp[r]) whose 16-bit column is >= h
cudaError_t launch_sell_split(int64_t rows, const int64_t* rp, const uint16_t* col16, int h,
                              int32_t* split, cudaStream_t st);

cudaError_t launch_momentum_resid(int64_t m, const float* r1, const float* r1lo, const float* r0,
                                  const float* r0lo, double beta, double* partials,
                                  unsigned* counter, double* scal, int grid, cudaStream_t st,
                                  const double* dbeta = nullptr);  // dbeta: device-side beta
cudaError_t launch_project(int64_t n, float* x, double lo, double hi, int grid, cudaStream_t st);
cudaError_t launch_gradient_map(int64_t n, const float* x, const float* g, double nu, double lo,
                                double hi, float* G, double* partials, unsigned* counter,
                                double* scal, int grid, cudaStream_t st);

struct TVArgs {
  int nx, ny, nzl;
  int64_t plane;
  int zg0, nzg;  // global z of local plane 0; global nz
  int zc;        // planes per work item (set by the launcher)
  double tau, alpha, lo, hi;
  // KIND_GRAD
  const float* w1;
  const float* w0;  // non-null: w = (1+wbeta) w1 - wbeta w0
  double wbeta;
  float* g_out;
  float* v_out;     // GRAD: optional; TRIAL: required
  const float* xp;  // BB reductions (with gp)
  const float* gp;
  double stop_step; // > 0: gradient-map reduction with this step
  // KIND_TRIAL
  const float* tx;
  const float* tg;
  const float* xo;  // mu_k reductions
  const float* xo_lo;  // extended iterates (SrcTrialX): lo part of xo
  float* v_lo_out;     // extended iterates: lo part of the written state
  double* partials;
  unsigned* counter;
  double* scal;     // 6 doubles
  // non-null (device-side control): [0] trial step s / momentum beta, [1] stop_step, [2] wbeta,
  // read by the kernel at launch instead of the values above.  The instantiation (which optional
  // reductions exist) is still chosen from the host-side fields, so a call site whose stop step is
  // decided on the device passes a positive placeholder stop_step.
  const double* dparam;
};

cudaError_t launch_tv_grad_plain(const TVArgs& a, const float* x, cudaStream_t st);
// x read in place with separate halo planes hlo (-1) and hhi (nzl)
cudaError_t launch_tv_grad_plain_h(const TVArgs& a, const float* x, const float* hlo,
                                   const float* hhi, cudaStream_t st);
cudaError_t launch_tv_grad_momentum(const TVArgs& a, const float* x1, const float* x0, double beta,
                                    cudaStream_t st);
cudaError_t launch_tv_trial(const TVArgs& a, const float* x, const float* g, double s,
                            cudaStream_t st);
// extended-precision iterates (hi + lo pairs; tv.cu SrcTrialX / SrcMomentumX): a.v_lo_out (and
// a.xo_lo with a.xo) required
// full: evaluate at the state hi + lo (with the A pass's lo gathers) instead of the hi part
cudaError_t launch_tv_trial_x(const TVArgs& a, const float* x, const float* x_lo, const float* g,
                              double s, cudaStream_t st, bool full);
cudaError_t launch_tv_grad_momentum_x(const TVArgs& a, const float* x1, const float* x1_lo,
                                      const float* x0, const float* x0_lo, double beta,
                                      cudaStream_t st, bool full);
cudaError_t launch_tv_grad_plain_x(const TVArgs& a, const float* x, const float* x_lo,
                                   cudaStream_t st);
cudaError_t launch_halo_fill_trial_x(const float* x, const float* x_lo, const float* g, double s,
                                     double lo, double hi, int64_t plane, int nzl, int n_lo,
                                     int n_hi, float* v, float* v_lo, cudaStream_t st,
                                     const double* dparam = nullptr);
cudaError_t launch_halo_fill_momentum_x(const float* x1, const float* x1_lo, const float* x0,
                                        const float* x0_lo, double beta, int64_t plane, int nzl,
                                        int n_lo, int n_hi, float* v, float* v_lo,
                                        cudaStream_t st, const double* dparam = nullptr);
int tv_num_blocks(int nx, int ny, int nzl);
int tv_set_grid(int num_sms);  // size the persistent stencil grid for the current device
cudaError_t launch_halo_fill_trial(const float* x, const float* g, double s, double lo, double hi,
                                   int64_t plane, int nzl, int n_lo, int n_hi, float* v,
                                   cudaStream_t st, const double* dparam = nullptr);
cudaError_t launch_halo_fill_momentum(const float* x1, const float* x0, double beta, int64_t plane,
                                      int nzl, int n_lo, int n_hi, float* v, cudaStream_t st,
                                      const double* dparam = nullptr);

cudaError_t build_transpose(int64_t m, int64_t n, int64_t nnz, const int64_t* rp,
                            const int32_t* col, const float* val, int64_t* rowT, int32_t* colT,
                            float* valT, int32_t* scratch_i32_n, int32_t* scratch_col,
                            float* scratch_val, int64_t* scratch_blocks, cudaStream_t st);

}  // namespace tvr

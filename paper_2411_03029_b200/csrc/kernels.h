// Launch wrappers for the sm_100a kernels (definitions in *_kernels.cu).
#pragma once

#include "common.cuh"
#include "level.cuh"

namespace tbf {

// ---- construction (id_kernels.cu)
size_t panel_smem_bytes(const LevelDesc& L);
size_t finish_smem_bytes(const LevelDesc& L);
void launch_gen_proxies(const LevelDesc& L, int* proxies, cudaStream_t st);
void launch_targets(const LevelDesc& L, const int* crank, const i64* cskel_off, const int* cskel, int* targets,
                    int* width, cudaStream_t st);
void launch_panel(const LevelDesc& L, const KSpec& ks, const int* proxies, const int* targets, const int* width,
                  double2* rpart, cudaStream_t st);
void launch_finish(const LevelDesc& L, double tol, double tie_eps, i64 max_rank, const double2* rpart,
                   const int* targets, const int* width, int* rank, int* sat, int* perm, int* skel_tmp,
                   double2* interp_tmp, double* gaps, cudaStream_t st);
void launch_compact(i64 nslots, i64 wmax, const int* rank, const int* width, const i64* skel_off,
                    const i64* interp_off, const int* skel_tmp, const double2* interp_tmp, int* skel, double2* interp,
                    cudaStream_t st);

// Generic batched column IDs of explicit matrices (column_id on the GPU):
// matrices are read from device memory instead of generated.
struct MatIdJob {
  i64 a_off;  // element offset of the m x n col-major matrix
  i64 m;
  int n;
  int pad;
};
void launch_matrix_panel(i64 njobs, const MatIdJob* jobs, const double2* A, i64 nparts, i64 rpp, int pr, i64 wmax,
                         double2* rpart, cudaStream_t st);

// ---- cores (core_kernels.cu)
struct PairDesc {
  i64 core_off;                 // element offset of the row-major R x C core
  int R, C;
  int rr[kMaxD], rc[kMaxD];     // per-mode ranks (rows: U side, cols: V side)
  i64 rs_off[kMaxD], cs_off[kMaxD];  // skeleton offsets (global 1-based ints)
  i64 work_off;                 // prefix of R*C over pairs (grid mapping)
};
void launch_cores(const KSpec& ks, i64 npairs, const PairDesc* pairs, i64 total_entries, const int* uskel,
                  const int* vskel, double2* cores, cudaStream_t st);

// ---- apply (apply_kernels.cu)
constexpr int kMaxTM = kMaxD + 1;  // tensor modes incl. n_v
struct MPStep {                     // one item of a batched block-diagonal mode product
  i64 in_off, out_off;
  i64 work_off;                     // prefix of output sizes (grid mapping)
  i64 total;                        // output elements
  i64 in_stride[kMaxTM], out_stride[kMaxTM];
  int ext[kMaxTM];                  // OUTPUT extents (contracted mode: Eout)
  int nd, mode, transpose, nblk;
  i64 blk_off;
};
struct Blk {
  i64 mat_off;  // element offset of the rows x cols col-major factor
  int rows, cols, in_start, out_start;
};
void launch_mode_product(i64 nitems, const MPStep* steps, i64 total_out, const Blk* blks, const double2* mats,
                         const double2* in, double2* out, cudaStream_t st);

struct GemvDesc {  // y(R x nv) = K(R x C, row-major) * x(C x nv)
  i64 core_off, x_off, y_off;
  int R, C;
  i64 cta_off;     // prefix of CTA counts
};
// cta_pair[i] = pair holding CTA i's first row; GemvDesc.cta_off = the pair's
// first global row
void launch_gemv(const int* cta_pair, const GemvDesc* d, i64 nctas, i64 total_rows, i64 rows_per_cta, int nv,
                 const double2* cores, const double2* x, double2* y, int max_c, cudaStream_t st);
int gemv_ctas_per_sm(int nv, int max_c);
// TMA bulk-copy pipelined variant (rows staged by cp.async.bulk into an SMEM ring)
void launch_gemv_tma(const int* cta_pair, const GemvDesc* d, i64 nctas, i64 total_rows, i64 rows_per_cta, int nv,
                     int stages, int stage_elems, int xcap, const double2* cores, const double2* x, double2* y,
                     cudaStream_t st);
size_t gemv_tma_smem_bytes(int stages, int stage_elems, int xcap);
int gemv_tma_max_pairs();

struct SumDesc {  // out[e] = sum_c in[c_off[c] + e], children in order
  i64 out_off, total, work_off;
  int nchild;
  int pad;
  i64 child_off[1 << kMaxD];
};
void launch_sum_children(i64 n, const SumDesc* d, i64 total, const double2* in, double2* out, cudaStream_t st);

// Fused box contraction (apply, one CTA per output box): the block-diagonal
// factor of every level splits the level into independent boxes; each box is
// out_box (+)= sum_terms in_box x_1 M_1 x_2 M_2 ... x_d M_d with all d modes
// applied in shared memory.  V/W: one term.  P (l >= 1): one term per child
// nu of p_nu, summed in ascending nu order.  U-bar / V-bar (l = 0) read / write
// the global tensors directly through strides.
struct BoxTerm {
  i64 in_off;
  i64 in_stride[kMaxTM];
  int in_ext[kMaxTM];
  i64 mat_off[kMaxD];
  int mrows[kMaxD], mcols[kMaxD];
};
struct BoxItem {
  i64 out_off;
  i64 out_stride[kMaxTM];
  int out_ext[kMaxTM];  // full box extents (last contracted mode: full, split by [last_lo, last_hi))
  int last_lo, last_hi;
  i64 term_off;
  int nterm, pad;
};
struct BoxLaunchInfo {
  int d, nv, transpose;
  int smem_elems_in, smem_elems_mat, smem_elems_a, smem_elems_b;
  int cs;              // thread-block cluster size: the last input mode is split over cs CTAs
  int smem_elems_acc;  // partial output box (cs > 1), reduced through DSMEM
};
void launch_box(i64 nitems, const BoxItem* items, const BoxTerm* terms, const BoxLaunchInfo& info,
                const double2* mats, const double2* in, double2* out, cudaStream_t st);
size_t box_smem_bytes(const BoxLaunchInfo& info);
void box_trace_enable(unsigned long long* buf);  // debug: per-CTA phase timestamps
int box_max_active_clusters(int cs, size_t smem);
// ordered child sums, one CTA per parent (SumDesc.work_off unused)
void launch_sum_parent(i64 nctas, const SumDesc* d, const int* cta_map, const double2* in, double2* out,
                       cudaStream_t st);

// ---- dense check (core_kernels.cu)
unsigned long long count_nonfinite(const double2* x, i64 n, cudaStream_t st);
void launch_dense_rows(const KSpec& ks, i64 nrows, const i64* rows, const double2* F, int nv, double2* out,
                       cudaStream_t st);

}  // namespace tbf

// Launch wrappers for the sm_100a kernels (definitions in *_kernels.cu).
#pragma once

#include "common.cuh"
#include "level.cuh"

namespace tbf {

// ---- FP64 roofline denominators (peak_kernels.cu)
void measure_fp64_peak(double* out);

// ---- construction (id_kernels.cu)
size_t panel_smem_bytes(const LevelDesc& L);
// panel rows and resident CTAs per SM of k_panel for a level of width wmax
void panel_shape(i64 wmax, i64 psize, int* pr, int* ctas_per_sm);
size_t finish_smem_bytes(const LevelDesc& L);
void launch_gen_proxies(const LevelDesc& L, int* proxies, cudaStream_t st);
void launch_targets(const LevelDesc& L, const int* crank, const i64* cskel_off, const int* cskel, int* targets,
                    int* width, cudaStream_t st);
void launch_panel(const LevelDesc& L, const KSpec& ks, const int* proxies, const int* targets, const int* width,
                  double2* rpart, cudaStream_t st);
void launch_finish(const LevelDesc& L, double tol, double tie_eps, i64 max_rank, const double2* rpart,
                   const int* targets, const int* width, int* rank, int* sat, int* perm, int* skel_tmp,
                   double2* interp_tmp, double* gaps, cudaStream_t st);
// closed-form narrow (w <= 2) column IDs of the separable DFT kernel
void launch_narrow_dft(const LevelDesc& L, const KSpec& ks, double tol, const int* crank, const i64* cskel_off,
                       const int* cskel, int* width, int* rank, int* sat, int* perm, int* skel_tmp, double2* interp_tmp,
                       double* gaps, cudaStream_t st);
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
// device-side bookkeeping: exclusive prefix sums of rank and rank * width per
// slot; middle-pair layout (same values as the host layout_pairs, world = 1)
void scan_slot_offsets(i64 n, const int* rank, const int* width, i64* skel_off, i64* interp_off, cudaStream_t st);
void layout_pairs_device(int d, i64 nmid, const int* urank, const i64* uskel_off, const int* vrank,
                         const i64* vskel_off, PairDesc* pairs, cudaStream_t st);

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
// first global row; CTA i owns rows [row_begin[i], row_begin[i+1]) (byte-balanced)
void launch_gemv(const int* cta_pair, const GemvDesc* d, i64 nctas, i64 total_rows, const i64* row_begin, int nv,
                 const double2* cores, const double2* x, double2* y, int max_c, cudaStream_t st);
int gemv_ctas_per_sm(int nv, int max_c);
// block-floating-point cores (fixed rate: 32-bit mantissas, one 16-bit
// exponent per 32 complex entries of a row; the ZFP role of PAPER.md Alg. 2)
void launch_bfp_compress(const long long* blk_prefix, i64 npairs, const GemvDesc* raw, const long long* q_off,
                         i64 total_blocks, const double2* cores, int2* q, short* ex, cudaStream_t st);
int gemv_bfp_ctas_per_sm(int max_c);
void launch_gemv_bfp(const int* cta_pair, const GemvDesc* d, i64 nctas, i64 total_rows, const i64* row_begin,
                     const int2* q, const short* ex, const double2* x, double2* y, int max_c, cudaStream_t st);
// TMA bulk-copy pipelined variant (rows staged by cp.async.bulk into an SMEM ring)
void launch_gemv_tma(const int* cta_pair, const GemvDesc* d, i64 nctas, i64 total_rows, const i64* row_begin, int nv,
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

// Fused box contraction (apply).  The block-diagonal factor of every level
// splits the level into independent boxes; each box is
//   out_box = in_box x_0 M_0 x_1 M_1 ... x_{d-1} M_{d-1}
// (M_k or M_k^T for the P/U side), all d modes applied on chip.  Modes are
// contracted d-1 first, 0 last; the cs CTAs of a box split the OUTPUT range
// of mode d-1, so they need no reduction.  in_box may be the ordered sum of
// nsum equally-shaped child tensors (P-level contributions, child c at
// in_off + c * sum_stride), summed while the input is staged.
struct BoxDesc {
  i64 in_off, out_off, sum_stride;
  i64 in_stride[kMaxTM], out_stride[kMaxTM];
  i64 mat_off[kMaxD];
  int ein[kMaxTM], eout[kMaxTM];  // per mode; entry d: nv
  int nsum, pad;
};
struct BoxLaunchInfo {
  int d, nv, transpose, cs;  // cs: CTAs per box (split of mode d-1's output)
  int amax;                  // max output rows of mode d-1 per CTA (template bucket: 2, 4 or 8)
  int stage;                 // 1: stage the whole input box in shared memory (cp.async)
  int smem_mat, smem_in, smem_t;  // elements: factors, staged input, intermediate buffer t0
  int smem_t1;                    // elements of intermediate buffer t1 (odd middle modes, staging table)
  int nt;                         // CTA size (256, or 128 for small boxes at up to 6 CTAs per SM)
  int mma;                        // FP64 tensor-core phases: 1 = unstaged mode d-1 (<= 16 input rows), 2 = and
                                  // mode 0 of the V / W side, 3 = and mode 0 of both sides, 4 = 2 and the V / W
                                  // side's middle modes (default)
  int afac;                       // 1: factor rows copied with cp.async (overlap the input staging)
  int split1;                     // 1: staged first mode splits a column's output rows over threads when columns are few
  int stream_out;                 // 1: mode 0 stores with the streaming hint (the output is the result tensor G)
  int tab_ok;                     // 1: every box's output span fits 32-bit column offsets (the mode-0 column table)
  int path;                       // compile-time variant of k_box for this launch (box_device.cuh: 0 any, 1 V / W
                                  // tensor-core box, 2 staged CUDA-core box)
};
void launch_box(i64 nitems, const BoxDesc* descs, const BoxLaunchInfo& info, const double2* mats,
                const double2* in, double2* out, cudaStream_t st);
size_t box_smem_bytes(const BoxLaunchInfo& info);
// d = 2 boxes as two register-tiled complex GEMMs, one CTA per box (box2_kernels.cu)
size_t box2_smem_bytes(int e0, int o0, int o1);
void launch_box2(i64 nitems, const BoxDesc* descs, const BoxLaunchInfo& info, size_t smem, const double2* mats,
                 const double2* in, double2* out, cudaStream_t st);
int box_ctas_per_sm(int nt, int stage, size_t smem);  // occupancy of k_box
// programmatic dependent launch for the apply kernels (env OIOBF_NO_PDL=1 disables)
bool pdl_enabled();

// ---- tiny-box apply engine (tiny_kernels.cu): one CTA per group of boxes that
// share data (V/W: the 2^d children tau of a parent, which all read the
// parent's output; P/U: the 2^d children nu summed into one parent), block
// geometry read from the level's slot arrays (no per-box descriptors)
constexpr int kTinyBox = 64;  // largest box (elements) the engine is chosen for
struct TinyGroup {
  i64 outer, pinner;  // V/W: (s, parent tau) [l = 0: (s, 0)];  P/U: (t, p_nu)
  i64 io_off;         // V/W: offset of the shared input tensor;  P/U: offset of the parent output
};
struct TinyLevelArgs {
  int side, l, d, nv, in_global, out_global;
  int nch;          // children per group (2^d, or 1 at l = 0)
  int threads;      // CTA size: the group's output count rounded up to a power of two, in [32, 256]
  i64 nin, nj, ngroups;
  i64 max_in;       // elements of staged input per group (shared memory)
  i64 fstride;      // factor elements per (child, mode) slot group; 0: factors read from global memory
  i64 xstride;      // P/U: staged input elements per child
  i64 ostride;      // V/W: output elements per child (thread map)
  i64 maxo;         // largest output extent of one mode (table size)
  i64 gstride[kMaxD + 1];  // strides of the global n^d x nv tensor (V0 input / U0 output)
};
size_t tiny_smem_bytes(const TinyLevelArgs& a);
// off_of[outer * nin + inner]: V/W child output offsets; P/U child input offsets
void launch_tiny_level(const TinyLevelArgs& a, const TinyGroup* groups, const i64* off_of, const int* rank,
                       const int* width, const i64* moff, const double2* mats, const double2* in, double2* out,
                       cudaStream_t st);
void launch_tiny_gemv(const GemvDesc* d, i64 npairs, i64 total_rows, int nv, const double2* cores, const double2* x,
                      double2* y, cudaStream_t st);

// ---- rank-one apply engine (r1_kernels.cu): every ID of rank 1, factor
// blocks 1 x W at slot * W, 1 x 1 cores at pair s * nmid + t; geometry implicit
struct R1LevelArgs {
  int side, l, d, W, nv, Lc;
  int nch;             // children per group (2^d at l >= 1, else 1)
  int gpb;             // V/W: groups per CTA; P/U: (group, block tuple) units per CTA
  int in_global;       // V/W l = 0: input is the n^d x nv tensor F
  int out_global;      // P/U l = 0: output is G
  int in_transposed;   // P/U l = Lc: input indexed by the pair s * nmid + t
  int core_mul;        // V/W l = Lc: multiply by the 1 x 1 core of pair s * nmid + t
  i64 n, nmid, mpm, mid;
  i64 nin, nj, njd;    // this level: inner multi-sets, blocks per mode, nj^d
  i64 pnin;            // groups per outer multi-set (parents)
  i64 ngroups;         // nmid * pnin
  i64 nunits;          // P/U: ngroups * njd
  i64 E, ED;           // V/W: input extent per mode and E^d; P/U: output extent and E^d
  int fblk, FS;        // factor elements per (outer, inner) slot group (d * nj * W); odd SMEM stride
  unsigned magic;      // ceil(2^32 / fblk): e / fblk as a multiply-high
  int lg_T;            // V/W: log2 consecutive tau per CTA; P/U cluster: log2 children per CTA
  int Pc;              // V/W: parents staged per CTA (max); P/U cluster: parents per cluster
  int XS;              // V/W: SMEM stride of a staged parent tensor (odd)
  int warp_tiles;      // V/W middle level: one warp per 32 consecutive tau (Pc = parents per warp
                       // tile); P/U levels >= 1: one warp per (group, block tuple) unit
  // log2 of the power-of-two extents above (n is a power of two)
  int lg_n, lg_mid, lg_nmid, lg_nin, lg_nj, lg_njd, lg_pnin, lg_nch, lg_E, lg_ED;
  // sharded (world > 1): this rank's 2^lg_nown outer multi-sets, local index i
  // -> middle multi-set own[i] (ascending); buffers, factor arenas and cores
  // are indexed by the LOCAL outer index, F / G slabs by own[i].  Unsharded:
  // lg_nown = lg_nmid, own = null (identity).
  int lg_nown;
  const int* own;
};
size_t r1_smem_bytes(const R1LevelArgs& a);
int r1_threads();
int r1_vthreads();
// column_id of explicit matrices wider than kMaxW (wide_id_kernels.cu): the
// reference's pivoted Householder QR in global memory, one CTA per matrix, on
// a work copy of the matrix (A is overwritten).  Per job: a_off / m / n, n_off
// = offset of its n-entry norm / perm / pos / skeleton arrays, i_off = offset
// of its interp (rank x n column-major, room for min(m, n) x n).
struct WideIdJob {
  i64 a_off, m, n_off, i_off, max_rank;
  int n, pad;
};
void launch_wide_ids(i64 njobs, const WideIdJob* jobs, double2* A, double* nrm, int* perm, int* pos, double tol,
                     int* rank, int* sat, int* skel, double2* interp, cudaStream_t st);
// sharded middle-level exchange of the rank-one engine: unpack = 0 packs the
// level-Lc V/W output into the send buffer, 1 unpacks the receive buffer into
// the level-Lc P/U input (off: the exchange offsets per pair t * nmid + s)
void launch_r1_exchange(const R1LevelArgs& a, int unpack, const long long* off, const double2* in, double2* out,
                        cudaStream_t st);
void launch_r1_level(const R1LevelArgs& a, const double2* fac, const double2* cores, const double2* in, double2* out,
                     cudaStream_t st);

// ---- dense check (core_kernels.cu)
unsigned long long count_nonfinite(const double2* x, i64 n, cudaStream_t st);
void launch_dense_rows(const KSpec& ks, i64 nrows, const i64* rows, const double2* F, int nv, double2* out,
                       cudaStream_t st);

}  // namespace tbf

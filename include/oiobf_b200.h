/* oiobf_b200.h — C ABI of the B200-native tensor-butterfly library
 * (paper_2411_03029_b200/libtbf_b200.so).
 *
 * This is the drop-in boundary under the reference's C++ construct/apply
 * interface (namespace oiobf, /root/reference/proj/include/oiobf/*.hpp).  Each
 * entry point names the reference function it replaces.  Conventions:
 *   - every function returns 0 on success, OIOBF_EINVAL for argument errors
 *     (the reference's std::invalid_argument, types.hpp:48-54) and
 *     OIOBF_ERUNTIME for CUDA failures; oiobf_last_error() gives the message
 *     (thread-local).  Exceptions never cross this boundary.
 *   - complex128 is interleaved (re, im) doubles, bit-compatible with
 *     std::complex<double>; tensors are first-mode-fastest (tensor.hpp:10-15);
 *     matrices column-major; indices 1-based where the reference API is.
 *   - host pointers are borrowed for the duration of the call; device memory is
 *     owned by opaque handles.
 *   - there is no CPU fallback: without a usable sm_100 device every compute
 *     entry point fails with OIOBF_ERUNTIME.
 */
#ifndef OIOBF_B200_H
#define OIOBF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OIOBF_OK 0
#define OIOBF_EINVAL 1
#define OIOBF_ERUNTIME 2

/* kernel catalog (BASELINE.json configs) */
#define OIOBF_KERNEL_GREEN 0   /* exp(-i kappa rho)/rho, plates (d=2) / cubes (d=3) */
#define OIOBF_KERNEL_DFT 1     /* exp(-2 pi i x.k), optional two-sided bit reversal  */
#define OIOBF_KERNEL_RADON2D 2 /* exp(2 pi i Phi(x,k))            */
#define OIOBF_KERNEL_RADON3D 3 /* exp(2 pi i (x.k + c|k|)), PAPER.md:644-646 (d=3)  */
#define OIOBF_KERNEL_NUDFT 4   /* type-2 NUDFT exp(2 pi i x^i.y^j), seeded random x^i */

/* ProxyMode (id.hpp:48) */
#define OIOBF_PROXY_ALL 0
#define OIOBF_PROXY_UNIFORM_RANDOM 1
#define OIOBF_PROXY_EVENLY_SPACED 2

/* POD kernel spec: replaces the opaque std::function in KernelEvaluator
 * (tensor.hpp:81-90) with a device-evaluable description. */
typedef struct oiobf_kernel_spec {
  int32_t kind;
  int32_t d;       /* modes per side, 1..6 */
  int64_t n;       /* points per mode (m_k = n_k = n) */
  int32_t bitrev;  /* DFT: two-sided per-mode bit reversal */
  uint32_t seed;   /* NUDFT: seed of the random target locations */
  double kappa;     /* Green: wavenumber */
  double offset[3]; /* Green: source-plane/cube offset added to y */
} oiobf_kernel_spec;

/* ProxyStrategy (id.hpp:50-55) */
typedef struct oiobf_proxy_strategy {
  int32_t mode;
  int32_t pad_;
  int64_t q;
  int64_t max_retries;
  int64_t row_cap;
} oiobf_proxy_strategy;

typedef struct oiobf_tbf oiobf_tbf; /* opaque device-resident TensorButterfly */

const char* oiobf_last_error(void);
/* device ordinal to use for subsequent calls of this thread (default 0) */
int oiobf_set_device(int device);
/* sm count, cc major/minor, total memory (bytes) of the current device */
int oiobf_device_info(int64_t out[4]);

/* ---- id-compress (id.hpp) ------------------------------------------------ */

/* Batched column_id (id.hpp:40, id.cpp:124-130): `batch` independent matrices,
 * A_b of shape m[b] x n[b] column-major at A + 2*a_off[b] (host, interleaved).
 * max_rank[b] < 0 means std::nullopt.  Outputs per matrix b (host):
 *   rank[b]; skeleton at skel + s_off[b] (n[b] slots, first rank used, 1-based
 *   sorted); interp (rank x n[b] col-major) at interp + 2*i_off[b] (room for
 *   n[b]*n[b]); perm (pivot order, 0-based, n[b] entries) at perm + s_off[b];
 *   saturated[b]; interp_max_abs[b].  ID of the proxy/unfolding matrix is
 *   computed on the GPU (TSQR + reference pivoting on R). */
int oiobf_column_id_batch(int64_t batch, const int64_t* m, const int64_t* n, const int64_t* a_off, const double* A,
                          double tol, const int64_t* max_rank, int64_t* rank, const int64_t* s_off, int64_t* skel,
                          const int64_t* i_off, double* interp, int64_t* perm, int32_t* saturated,
                          double* interp_max_abs);

/* select_proxies_count (id.cpp:155-185), bit-exact; out has room for extent. */
int oiobf_select_proxies_count(int64_t extent, int64_t count, int32_t mode, uint64_t seed, int64_t* out,
                               int64_t* out_count);

/* derive_seed (rng.hpp:39-47) */
uint64_t oiobf_derive_seed(uint64_t seed, const uint64_t* tags, int32_t ntags);

/* subtensor_at (tensor.cpp:249-266): K(rows, cols) over explicit per-mode
 * index lists (2d lists concatenated, counts[2d]), evaluated on the GPU;
 * out = prod(counts) complex, first mode fastest. */
int oiobf_subtensor_at(const oiobf_kernel_spec* spec, const int64_t* counts, const int64_t* lists, double* out);

/* mode_product_blockdiag (tensor.cpp:136-166) on the GPU.  t: nmodes-mode
 * tensor of `shape`; blocks concatenated col-major with shapes (br[b], bc[b]). */
int oiobf_mode_product_blockdiag(int32_t nmodes, const int64_t* shape, const double* t, int32_t mode, int32_t nb,
                                 const int64_t* br, const int64_t* bc, const double* blocks, int32_t transpose,
                                 double* out);

/* ---- tensor-butterfly ----------------------------------- */

/* tbf_construct(eval, L, tol, proxies, seed) (PAPER Alg. 1).
 * L even, n = C_b * 2^L.  Factors and cores stay in device memory. */
int oiobf_tbf_construct(const oiobf_kernel_spec* spec, int32_t L, double tol, const oiobf_proxy_strategy* proxies,
                        uint64_t seed, oiobf_tbf** out);
int oiobf_tbf_destroy(oiobf_tbf* h);

/* tbf_contract(bf, F) (PAPER Alg. 2) with host buffers:
 * F, G: n^d x nv complex, first mode fastest.  Includes H2D/D2H copies. */
int oiobf_tbf_contract(oiobf_tbf* h, const double* F, double* G, int64_t nv);

/* Stream-ordered tbf_contract with PINNED host buffers: enqueues H2D(F) ->
 * contraction -> D2H(G) on the handle's copy / compute streams, makes `stream`
 * (cudaStream_t, NULL = legacy default) wait for the result, and returns.
 * Two calls per (handle, nv) can be in flight with their own device staging,
 * so the H2D of one call overlaps the contraction of the previous one and the
 * D2H of the one before (PCIe is full duplex).  F must stay unmodified and G
 * unread until `stream` reaches this point.  Pageable F or G: error. */
int oiobf_tbf_contract_async(oiobf_tbf* h, const double* F, double* G, int64_t nv, void* stream);

/* Same with device buffers (double2*), enqueued on `stream` (cudaStream_t,
 * NULL = legacy default).  Replays a captured CUDA graph after the first call
 * for a given (nv, F, G, stream). */
int oiobf_tbf_contract_device(oiobf_tbf* h, const void* dF, void* dG, int64_t nv, void* stream);

/* tbf_memory: bytes of V, W, U, P, cores (out[5]). */
// TBF1 serialization: self-describing little-endian file
// (header, factor blocks in canonical tree order, cores, FNV-1a checksum);
// save -> load round trips are bit-exact.  load returns a new handle on the
// current device (oiobf_tbf_destroy it).
int oiobf_tbf_save(const oiobf_tbf* h, const char* path);
int oiobf_tbf_load(const char* path, oiobf_tbf** out);

// Apply engine: 0 auto (the rank-one engine when every ID has rank 1 and the
// leaf size is <= 2, e.g. the two-sided bit-reversed DFT; else the tiny-box
// engine when every box has <= 64 elements and there are >= 2^20 middle pairs;
// else the fused-box engine), 1 the fused-box engine, 2 the tiny-box engine,
// 4 the rank-one engine (OIOBF_EINVAL when the factorization is not eligible;
// 3, the round-1 dataflow engine, was removed).  Changing it drops cached plans.
/* Core storage for the apply: 0 = FP64 (exact, default); 1 = block floating
 * point -- the role ZFP plays in PAPER.md Alg. 2 ("ZFP decompress K(tbar,
 * sbar)"): per 32 entries of a core row one 16-bit exponent, per component a
 * 32-bit mantissa (8.06 instead of 16 bytes per entry; every entry within
 * 2^-31 of its block's largest component, ~5e-10 relative), decoded in the
 * core GEMV (n_v = 1).  The FP64 cores stay resident; the rank-one engine
 * (1 x 1 cores) refuses format 1. */
int oiobf_tbf_set_core_format(oiobf_tbf* h, int32_t format);
int oiobf_tbf_set_apply_engine(oiobf_tbf* h, int32_t engine);
// engine in use: 1 box, 2 tiny, 4 rank-one
int oiobf_tbf_apply_engine(oiobf_tbf* h, int32_t* engine);

int oiobf_tbf_memory(const oiobf_tbf* h, int64_t out[5]);

/* info[0..9]: d, n, L, Lc, nmid, total_slots, total_skel, total_interp,
 * total_core, total_perm (sizes for oiobf_tbf_export). */
int oiobf_tbf_info(const oiobf_tbf* h, int64_t info[10]);

/* Flat export in canonical slot order: V/W levels 0..Lc then
 * U/P levels 0..Lc; per slot rank, ncols, rows; skeletons (global 1-based),
 * interps (rank x ncols col-major), pivot orders; cores per pair p = s*nmid+t
 * in the reference's matricized column-major layout; r_est per (side, level).
 * Any output pointer may be NULL to skip it. */
int oiobf_tbf_export(const oiobf_tbf* h, int64_t* ranks, int64_t* ncols, int64_t* rows, int64_t* skel,
                     double* interp, int64_t* perm, double* cores, int64_t* core_rows, int64_t* core_cols,
                     int64_t* r_est);
/* Cores of selected middle pairs (sorted p = s * nmid + t) for block-wise
 * checks: core_rows / core_cols for all pairs (core_cols = 0 when not
 * selected), selected cores packed in pair order, column-major. */
int oiobf_tbf_export_cores(const oiobf_tbf* h, int64_t nsel, const int64_t* sel, double* cores, int64_t* core_rows,
                           int64_t* core_cols);

/* Robustness diagnostic: non-finite entries per (side, level) interp arena
 * (out[2q], with the level's max rank in out[2q+1]) and in the cores
 * (out[4*(Lc+1)]). */
int oiobf_tbf_check_finite(oiobf_tbf* h, int64_t* out);

/* Construction timing breakdown (ms): [proxies+targets, panel TSQR, finish,
 * compaction, cores, total] accumulated over levels. */
int oiobf_tbf_timings(const oiobf_tbf* h, double out[6]);

/* Apply-plan statistics for roofline accounting: out[0] = algorithmic bytes of
 * one contraction at nv=1 (16 * (2 n^d + sum|V,W,U,P| + sum|cores|)),
 * out[1] = core bytes, out[2] = number of kernel launches per contraction,
 * out[3] = complex MACs per contraction at nv=1. */
int oiobf_tbf_plan_stats(oiobf_tbf* h, int64_t out[4]);

/* Per-kernel timing of one device contraction (ms per launch group):
 * out[0] = factor steps (V/W), out[1] = core GEMV, out[2] = P/U steps, out[3] = total.
 * Timed with CUDA events on `stream`, averaged over `reps` contractions. */
int oiobf_tbf_profile_contract(oiobf_tbf* h, const void* dF, void* dG, int32_t reps, void* stream, double out[4]);
/* Cold-L2 timing of the core-contraction phase alone (flush buffer of
 * flush_bytes overwritten before each of reps launches); *out = mean ms. */
int oiobf_tbf_profile_core_cold(oiobf_tbf* h, const void* dF, void* dG, int32_t reps, void* stream, void* flush,
                                int64_t flush_bytes, double* out);
/* FP64 peaks of the current device: out[0] DFMA TFLOP/s, out[1] DMMA
 * (mma.sync.m8n8k4.f64) TFLOP/s, out[2] SM count, out[3] SM clock MHz. */
int oiobf_fp64_peak(double out[4]);

/* K-check: direct dense sums G(i, v) = sum_j K(i, j) F(j, v) on the GPU for
 * `nrows` sampled output flat indices (first mode fastest); F host n^d x nv. */
int oiobf_dense_rows(const oiobf_kernel_spec* spec, const double* F, int64_t nv, int64_t nrows,
                     const int64_t* rows_flat, double* out);

/* ---- sharded (multi-GPU) construction and apply, SURVEY §8(e) -------------
 * One process per GPU.  Rank r owns the middle multi-sets o with owner(o) ==
 * r on both sides -- o % world by default, or the map given to
 * oiobf_tbf_shard_set_owners (byte-balanced ownership: the same map on every
 * rank, set right after oiobf_tbf_shard_begin).  It builds the V/W IDs of its column multi-sets s, the
 * U/P IDs of its row multi-sets t, and the cores of the pairs (t, s) with s
 * owned.  The caller performs the collectives (torch.distributed / NCCL):
 *   1. oiobf_tbf_shard_begin, then for each side and level l = 0..Lc:
 *      oiobf_tbf_shard_level(r_est) with r_est = max(8, all-reduce-max of the
 *      local max ranks of the previous levels of that side)
 *   2. oiobf_tbf_umid_export -> sum all-reduce -> oiobf_tbf_umid_import
 *      (row skeletons of every t at level Lc; builds the owned cores)
 *   3. oiobf_tbf_set_exchange(send / receive offsets of every G_{t,s} block)
 *   4. apply: oiobf_tbf_contract_phase(1, F, send) ; all-to-all(send -> recv) ;
 *      oiobf_tbf_contract_phase(2, recv, G).
 */
int oiobf_tbf_shard_begin(const oiobf_kernel_spec* spec, int32_t L, double tol, const oiobf_proxy_strategy* proxies,
                          uint64_t seed, int32_t rank, int32_t world, oiobf_tbf** out);
/* owners[o] in [0, world) for every middle multi-set o (nmid entries); before the first level */
int oiobf_tbf_shard_set_owners(oiobf_tbf* h, const int32_t* owners);
int oiobf_tbf_shard_level(oiobf_tbf* h, int32_t side, int32_t level, int64_t r_est, int64_t* local_max_rank);
int oiobf_tbf_umid_info(oiobf_tbf* h, int64_t out[2]);
int oiobf_tbf_umid_export(oiobf_tbf* h, int64_t* ranks, int32_t* skel, int64_t wpad);
int oiobf_tbf_umid_import(oiobf_tbf* h, const int64_t* ranks, const int32_t* skel, int64_t wpad);
int oiobf_tbf_set_exchange(oiobf_tbf* h, const int64_t* send_off, const int64_t* recv_off, int64_t send_elems,
                           int64_t recv_elems);
int oiobf_tbf_contract_phase(oiobf_tbf* h, int32_t phase, const void* dIn, void* dOut, int64_t nv, void* stream);

// Fused exchange (replaces the all-to-all between the phases): the phase-1 core
// GEMV stores every block G_{t,s} straight into the receive buffer of the
// owner of t (peer memory over NVLink, mapped with oiobf_ipc_open).
// recv_base[par * world + q] = device address (in this process) of rank q's
// receive buffer of parity par (0/1: consecutive steps alternate, so a step's
// stores never overwrite a buffer a peer is still reading); peer_off[t * nmid
// + s] = element offset (n_v = 1) of block (t, s) in its owner's receive
// buffer, for the pairs whose s this rank owns (-1 elsewhere); nv_max bounds
// n_v.  Phase 1 is then called with dOut = recv_base[par * world + rank].
// recv_base = NULL returns to the send buffer + all-to-all path.
int oiobf_tbf_set_peer_exchange(oiobf_tbf* h, const int64_t* peer_off, const uint64_t* recv_base, int32_t world,
                                int64_t nv_max);
// device buffers with a stable base address (for IPC) and CUDA IPC handles
int oiobf_device_alloc(int64_t bytes, void** out);
int oiobf_device_free(void* p);
int oiobf_ipc_handle(void* p, uint8_t handle[64]);
int oiobf_ipc_open(const uint8_t handle[64], void** out);
int oiobf_ipc_close(void* p);
// copies between any two of host / this device / a peer device (UVA,
// cudaMemcpyDefault; synchronous), and a device-wide synchronize of the
// calling thread's device -- the plumbing of the in-process multi-device
// driver in include/oiobf/sharded.hpp (one handle per device, peer copies over
// NVLink for the exchange)
int oiobf_memcpy(void* dst, const void* src, int64_t bytes);
// Owned-slab copies of a sharded handle (stream-ordered, strided DMA, no
// staging): dir 0 copies the input sub-tensors F(s) of the middle column
// multi-sets s this rank owns from host F to device dF (what phase 1 reads);
// dir 1 copies the output sub-tensors G(t) of the owned row multi-sets t from
// device dG to host G (what phase 2 wrote).  F / G: n^d x nv, first mode
// fastest; host buffers should be pinned for the copies to be asynchronous.
int oiobf_tbf_copy_owned(oiobf_tbf* h, int32_t dir, const void* src, void* dst, int64_t nv, void* stream);
int oiobf_synchronize(void);

#ifdef __cplusplus
}
#endif

#endif /* OIOBF_B200_H */

/*
 * corutv_b200.h — C-ABI of the B200-native (sm_100a) CoR-UTV / ALM-CoRUTV
 * hot path.  Plain pointers and sizes only; all matrices are row-major
 * (C-order) float64, exactly as the reference's numpy arrays
 * (/root/reference/pkg/src/corutv/dense.py:4-7).  Matrix pointers are DEVICE
 * pointers unless the parameter name ends in `_host`; every call is
 * asynchronous on the handle's stream unless it returns a host scalar.
 *
 * Each entry point names the reference interface it replaces
 * (file:line under /root/reference/pkg/src/corutv/).  The Python host layer
 * (paper_1906_04572_b200/) binds these with ctypes; INTEGRATION.md shows the
 * binding a maintainer adds on the reference side.
 */
#ifndef CORUTV_B200_H
#define CORUTV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes (the Python shim maps them to the reference's exceptions). */
enum corutv_status {
  CORUTV_OK = 0,
  CORUTV_ERR_SHAPE = 1,      /* ValueError: "rows >= cols", "exceeds", bad dims (sketch.py:93-98,192-193) */
  CORUTV_ERR_NONFINITE = 2,  /* ValueError: "contains non-finite entries" (dense.py:48-49) */
  CORUTV_ERR_CUDA = 3,       /* CUDA runtime/launch failure (CorutvError) */
  CORUTV_ERR_COMM = 4,       /* collective failure in the row-sharded path (CorutvError) */
  CORUTV_ERR_CONVERGENCE = 5,/* iteration cap hit (ConvergenceError, errors.py:8-18) */
  CORUTV_ERR_ARG = 6,        /* invalid argument (ValueError) */
  CORUTV_ERR_NOMEM = 7,      /* device allocation failed (CorutvError) */
  CORUTV_ERR_IO = 8          /* the row-reader callback failed (OSError) */
};

/* Row reader for streamed input: fill dst (rows x n, leading dimension ld,
 * pinned host memory owned by the library) with rows [row0, row0 + rows)
 * of the matrix; return 0 on success. */
typedef int (*corutv_read_rows_fn)(void* user, int64_t row0, int64_t rows, double* dst, int64_t ld);

enum corutv_variant { CORUTV_EXACT_D = 0, CORUTV_APPROX_D = 1 }; /* sketch.py:52-55 */

typedef struct corutv_handle corutv_handle;

/* Sum-allreduce of `count` float64 values in place on `stream`; returns 0 on
 * success.  Installed for the row-sharded (multi-GPU) path: the host binds it
 * to NCCL (torch.distributed) or to any transport.  NULL = single GPU. */
typedef int (*corutv_allreduce_fn)(void* user, double* buf, int64_t count, void* stream);

/* Library / device handle: owns a growable device workspace and the stream
 * (a cudaStream_t, or NULL for the legacy default stream). */
int corutv_create(int device, void* stream, corutv_handle** out);
void corutv_destroy(corutv_handle* h);
/* Rebind the handle to `stream`; the new stream is ordered after the work
 * already queued on the old one (it still reads the handle's workspace). */
int corutv_set_stream(corutv_handle* h, void* stream);
const char* corutv_last_error(const corutv_handle* h);
int corutv_version(void);

/* Row-sharded mode: this rank owns `m_local` consecutive rows of the global
 * matrix; sketches over the column space are combined with `fn`
 * (SURVEY §8e).  world == 1 (or fn == NULL) restores single-GPU mode. */
int corutv_set_comm(corutv_handle* h, corutv_allreduce_fn fn, void* user, int rank, int world);

/* Native NCCL data plane of the row-sharded mode: every
 * exchange point (the n x ell sketch sum, the Gram of the row-sharded Q1
 * sketch, the ell x ell core, the spectral norm's Gram and n x b block, the
 * ALM scalars) is an ncclAllReduce enqueued by the library on the handle's
 * stream -- no host callback, no host synchronisation of its own.
 *   corutv_nccl_unique_id     : rank 0 creates the 128-byte ncclUniqueId
 *                               (the host layer broadcasts it);
 *   corutv_nccl_comm_create   : every rank joins (ncclCommInitRank on
 *                               `device`); the caller owns the ncclComm_t;
 *   corutv_nccl_comm_destroy  : ncclCommDestroy;
 *   corutv_set_nccl           : attach a communicator to a handle for the
 *                               following calls (NULL detaches).
 * NCCL (libnccl.so.2) is resolved at run time.  A one-rank communicator
 * runs the sharded code path on one GPU.  corutv_set_comm detaches it. */
int corutv_nccl_unique_id(unsigned char* id_out);
int corutv_nccl_comm_create(int device, const unsigned char* id, int rank, int world, void** comm_out);
int corutv_nccl_comm_destroy(void* nccl_comm);
int corutv_set_nccl(corutv_handle* h, void* nccl_comm, int rank, int world);

/* Row-sharded mode: the global row count of the matrices of the following
 * calls (the same on every rank), so no call needs a row-count collective
 * and host sync.  0 = unknown (one allreduce per call).  Reset by
 * corutv_set_comm. */
int corutv_set_global_rows(corutv_handle* h, int64_t m_global);

/* CoR-UTV: replaces corutv(a, cfg, counter) — sketch.py:182-208, including
 * _power_sketch (sketch.py:166-179), householder_qr of both sketches
 * (dense.py:132-149; here a backward-stable adaptive shifted CholeskyQR),
 * compression (sketch.py:155-158 exact-d / sketch.py:203 approx-d), qrcp
 * (dense.py:152-192) and the lift (sketch.py:205-207).
 *   a      : m x n, leading dimension lda (in the sharded mode: the local
 *            m x n row block; the global row count is the sum over ranks)
 *   omega  : n x ell Gaussian test matrix (gaussian_matrix, sketch.py:63-68)
 *   u      : m x ell (ld ell)    t : ell x ell upper triangular (ld ell)
 *   v      : n x ell (ld ell)    perm : ell int64 (nullable)
 *   passes_host : incremented by the number of data sweeps (PassCounter,
 *                 sketch.py:126-163): 2q+3 exact-d, 2q+2 approx-d (nullable)
 * Synchronises the stream before returning (status depends on device flags). */
int corutv_decompose(corutv_handle* h, const double* a, int64_t m, int64_t n, int64_t lda,
                     int ell, int q_power, int variant, const double* omega, double* u, double* t,
                     double* v, int64_t* perm, int64_t* passes_host);

/* Same, with the Gaussian test matrix drawn on the device from the PCG64
 * state numpy's PCG64(seed) starts from: pcg_state = {state_hi, state_lo,
 * inc_hi, inc_lo} (np.random.PCG64(seed).state, i.e. SeedSequence-expanded on
 * the host).  Omega is bit-identical to gaussian_matrix(n, ell, seed)
 * (sketch.py:63-68). */
int corutv_decompose_seeded(corutv_handle* h, const double* a, int64_t m, int64_t n, int64_t lda,
                            int ell, int q_power, int variant, const uint64_t* pcg_state, double* u,
                            double* t, double* v, int64_t* perm, int64_t* passes_host);

/* CoR-UTV truncated for the ALM thresholding step (rpca.py:122-132,
 * _truncate_utv): r = #(|diag T| > delta) is returned in *r_host.  The QRCP
 * stops once the largest remaining (downdated) column norm is below delta
 * (with a 1e-3 margin for the downdate error), so every diagonal entry that
 * can exceed delta is computed and counted, as the reference counts the
 * whole diagonal even where it is slightly non-monotone; U[:, :r], T's rows
 * up to the last step taken (later rows zeroed), V and perm are formed.
 * Omega from `omega` (n x ell, device) or, if NULL, drawn from pcg_state as
 * corutv_decompose_seeded.  Any ell <= min(m, n). */
int corutv_decompose_truncated(corutv_handle* h, const double* a, int64_t m, int64_t n, int64_t lda,
                               int ell, int q_power, int variant, const double* omega,
                               const uint64_t* pcg_state, double delta, double* u, double* t,
                               double* v, int64_t* perm, int64_t* passes_host, int* r_host);

/* corutv(a, cfg) for a HOST-resident A (sketch.py:182-208 with the
 * as_matrix H2D of a numpy input, dense.py:41-50): A (m x n, lda_host;
 * pinned or pageable) is copied into the caller's device buffer a_dev
 * (m x ld_dev, 16-byte aligned, ld_dev even) in ~1 GiB row chunks on a copy
 * stream, and the first sketch sweep C1 = A Omega consumes each chunk as it
 * lands.  Results are bit-identical to corutv_decompose on the same device
 * buffer.  Omega from `omega` (device) or, if NULL, from pcg_state. */
int corutv_decompose_host(corutv_handle* h, const double* a_host, int64_t m, int64_t n,
                          int64_t lda_host, double* a_dev, int64_t ld_dev, int ell, int q_power,
                          int variant, const double* omega, const uint64_t* pcg_state, double* u,
                          double* t, double* v, int64_t* perm, int64_t* passes_host);

/* Economy SVD by one-sided Jacobi (dense.py:357-376, tol 1e-14, 100
 * sweeps; zero singular values get the deterministic orthonormal completion
 * of dense.py:285-310): u (m x k), sigma (k, descending), v (n x k), k =
 * min(m, n) <= 16384, all device row-major.  CORUTV_ERR_CONVERGENCE if the
 * sweeps do not converge. */
int corutv_jacobi_svd(corutv_handle* h, const double* a, int64_t m, int64_t n, int64_t lda,
                      double* u, double* sigma, double* v);

/* jacobi_svd(a, tol, max_sweeps, v_init) (dense.py:313-376): the sweeps
 * start from A_tall v_init, A_tall = a (m >= n) or a' (m < n), and the right
 * factor of A_tall is v_init times the rotations.  v_init: k x k device
 * (ld ldvi), orthonormal, or NULL (cold start).  tol / max_sweeps: the
 * stopping rule of dense.py:223-282 (reference defaults 1e-14 / 100).
 * Replaces _jacobi_svd_tall's v_init branch dense.py:315-321, 352-353. */
int corutv_jacobi_svd_warm(corutv_handle* h, const double* a, int64_t m, int64_t n, int64_t lda,
                           const double* v_init, int64_t ldvi, double tol, int max_sweeps,
                           double* u, double* sigma, double* v);

/* Singular value thresholding step of the InexactALM baseline
 * (_svt_warm rpca.py:146-158): warm-started Jacobi SVD of b (m x n), then
 * kept = max(sigma - delta, 0) (k), t = diag(kept) (k x k, ld k),
 * *r_host = #(kept > 0), capped at `cap` when cap >= 0.  u (m x k), v
 * (n x k) as corutv_jacobi_svd_warm, so u[:, :r] (t[:r, :] v') is the
 * thresholded matrix (feed u, t, v, ell = k, r to corutv_alm_update /
 * corutv_lowrank); v is the next call's v_init for square b. */
int corutv_svt(corutv_handle* h, const double* b, int64_t m, int64_t n, int64_t ldb,
               double delta, int cap, const double* v_init, int64_t ldvi, double* u,
               double* kept, double* v, double* t, int* r_host);

/* sor_svd (sketch.py:244-262): the corutv pipeline (power sketch, both
 * sketch QRs, exact or approximate compression) finished by a one-sided
 * Jacobi SVD of the l x l core (dense.py:357-376) instead of the QRCP:
 * u (m x l) = Q1 Uc, sigma (l, descending), v (n x l) = Q2 Vc, all device.
 * Omega from `omega` (n x l, device) or, if NULL, from pcg_state.  Requires
 * m >= n. */
int corutv_sor_svd(corutv_handle* h, const double* a, int64_t m, int64_t n, int64_t lda, int ell,
                   int q_power, int variant, const double* omega, const uint64_t* pcg_state,
                   double* u, double* sigma, double* v, int64_t* passes_host);

/* tsr_svd (sketch.py:220-241): two-sided randomized SVD from one
 * algorithmic pass: y = A psi (psi n x l), z = A' phi (phi m x l), Q1 =
 * orth(y), Q2 = orth(z), core = (Q1' y) pinv(Q2' psi), Jacobi SVD of the
 * core, lifted.  psi / phi given (device) or drawn from pcg_psi / pcg_phi
 * (the reference uses seed and seed + 0x9E3779B9 mod 2^64).  Any m, n with
 * l <= min(m, n).  *passes_host += 1 (the reference's fused-sweep count). */
int corutv_tsr_svd(corutv_handle* h, const double* a, int64_t m, int64_t n, int64_t lda, int ell,
                   const double* psi, const uint64_t* pcg_psi, const double* phi,
                   const uint64_t* pcg_phi, double* u, double* sigma, double* v,
                   int64_t* passes_host);

/* corutv of a matrix that is never resident in host memory (an out-of-core
 * file): the library pulls ~1 GiB row chunks through
 * read_rows into two pinned staging buffers, copies each to the caller's
 * device buffer a_dev (m x ld_dev, 16-byte aligned, ld_dev even) on a copy
 * stream and runs the first sketch sweeps on each chunk as it lands, as
 * corutv_decompose_host does; the read of chunk c+1 overlaps the copy and
 * the sweeps of chunk c.  Bit-identical to corutv_decompose on a_dev. */
int corutv_decompose_stream(corutv_handle* h, corutv_read_rows_fn read_rows, void* user, int64_t m,
                            int64_t n, double* a_dev, int64_t ld_dev, int ell, int q_power,
                            int variant, const double* omega, const uint64_t* pcg_state,
                            double* u, double* t, double* v, int64_t* perm, int64_t* passes_host);

/* sor_svd / tsr_svd of a HOST-resident A, streamed as corutv_decompose_host
 * does: A (m x n, lda_host) is copied into a_dev (m x ld_dev, 16-byte
 * aligned, ld_dev even) in row chunks overlapped with the first products
 * (for tsr_svd both y = A psi and z = A' phi consume each chunk as it
 * lands: one pass over the host data).  Bit-identical to the resident
 * calls on a_dev. */
int corutv_sor_svd_host(corutv_handle* h, const double* a_host, int64_t m, int64_t n, int64_t lda_host,
                        double* a_dev, int64_t ld_dev, int ell, int q_power, int variant,
                        const double* omega, const uint64_t* pcg_state, double* u, double* sigma,
                        double* v, int64_t* passes_host);
int corutv_tsr_svd_host(corutv_handle* h, const double* a_host, int64_t m, int64_t n, int64_t lda_host,
                        double* a_dev, int64_t ld_dev, int ell, const double* psi,
                        const uint64_t* pcg_psi, const double* phi, const uint64_t* pcg_phi,
                        double* u, double* sigma, double* v, int64_t* passes_host);

/* Host -> device copy of a row-major matrix (the as_matrix upload of a
 * numpy input, dense.py:41-50) in ~1 GiB row chunks on the copy stream:
 * pinned sources by DMA, pageable ones through pinned staging filled by a
 * multi-threaded host copy.  Returns after the copy completed. */
int corutv_upload(corutv_handle* h, const double* host, int64_t rows, int64_t cols, int64_t ld_host,
                  double* dev, int64_t ld_dev);

/* Device -> host copy of a row-major matrix (factors or L, S returned to a
 * numpy caller) through two pinned staging slots: the D2H of one chunk
 * overlaps the multi-threaded copy-out of the previous one.  Ordered after
 * the work queued on the handle's stream; returns when the data is in host. */
int corutv_download(corutv_handle* h, const double* dev, int64_t rows, int64_t cols, int64_t ld_dev,
                    double* host, int64_t ld_host);

/* np.random.Generator(PCG64(seed)).standard_normal((rows, cols)) into out
 * (row-major, ld) on the device, bit-identical (gaussian_matrix,
 * sketch.py:63-68).  One stream synchronisation (tail-sample readback);
 * the result is ordered on the handle's stream. */
int corutv_gaussian(corutv_handle* h, const uint64_t* pcg_state, int64_t rows, int64_t cols,
                    double* out, int64_t ld);

/* Fused ALM update, rpca.py:211-216 with L = U[:, :r] (T[:r,:] V')
 * (rpca.py:129) formed tile-by-tile and never stored:
 *   g  = (M - L) + Y/mu ;  S = sign(g) max(|g| - lam/mu, 0)
 *   Z  = (M - L) - S    ;  Y <- Y + mu Z
 *   G' = (M - S) + Y/mu_next   (the next iteration's input, rpca.py:208)
 * and returns zeta2 = sum Z^2 and nnz = #(|S| > 1e-12) (rpca.py:215-216).
 * m_mat, s, y, g_next: rows x cols (ld cols); u: rows x ell (ld ell);
 * t: ell x ell; v: cols x ell.  r in [0, ell]. */
int corutv_alm_update(corutv_handle* h, const double* m_mat, double* s, double* y, double* g_next,
                      int64_t rows, int64_t cols, const double* u, const double* t,
                      const double* v, int ell, int r, double mu, double lam_over_mu,
                      double mu_next, double* zeta2_host, int64_t* nnz_host);

/* L = U[:, :r] (T[:r, :] V')  — rpca.py:122-132 (_truncate_utv), written out. */
int corutv_lowrank(corutv_handle* h, const double* u, const double* t, const double* v,
                   int64_t rows, int64_t cols, int ell, int r, double* l_out);

/* corutv_lowrank_error with only the leading r rows of T kept:
 * |A - U[:, :r] (T[:r, :] V')|_F, the truncated-UTV error of bench.py's
 * "utv-approx" method (bench.py:219-222).  0 <= r <= ell. */
int corutv_lowrank_error_rank(corutv_handle* h, const double* a, int64_t m, int64_t n, int64_t lda,
                              const double* u, const double* t, const double* v, int ell, int r,
                              double* out_host);

/* Column-pivoted QR of an m x n device matrix (qrcp, dense.py:152-192:
 * Businger-Golub pivoting on downdated column norms with exact refresh,
 * first-index ties): q (m x k, ld ldq), r (k x n upper, ld ldr), perm (n)
 * with a[:, perm] = q r, k = min(m, n).  Square cores up to 640 run in one
 * CTA or a thread-block cluster; anything else in one cooperative grid
 * launch with the matrix in L2 (m + n/2 up to ~28000). */
int corutv_qrcp_mn(corutv_handle* h, const double* a, int64_t m, int64_t n, int64_t lda, double* q,
                   int64_t ldq, double* r, int64_t ldr, int64_t* perm);

/* Square case of corutv_qrcp_mn (q, r n x n, ld n): the harness's
 * deterministic "qrcp" method (bench.py:151-152, 208-211). */
int corutv_qrcp(corutv_handle* h, const double* a, int64_t n, int64_t lda, double* q, double* r,
                int64_t* perm);

/* |A|_2 by block power iteration — dense.py:405-442 (b = min(24, n),
 * disjoint-support start, stop when |est - prev| <= 0.02 tol est).
 * Matrices with min(m, n) <= 64 use the one-sided Jacobi path
 * (dense.py:414-415). */
int corutv_spectral_norm(corutv_handle* h, const double* a, int64_t m, int64_t n, int64_t lda,
                         double tol, int max_iter, double* out_host, int* iters_host);

/* Singular values (descending) of an m x n matrix — dense.py:379-387
 * (one-sided Jacobi, tol 1e-14, <= 100 sweeps; one CTA when the columns fit
 * shared memory, else the cooperative grid), min(m, n) <= 16384.
 * sig: min(m,n) doubles. */
int corutv_singular_values(corutv_handle* h, const double* a, int64_t m, int64_t n, int64_t lda,
                           double* sig);

/* Number of non-finite entries of an m x n matrix (as_matrix's check,
 * dense.py:48-49), this rank only; *count_host receives it. */
int corutv_count_nonfinite(corutv_handle* h, const double* a, int64_t m, int64_t n, int64_t lda,
                           int64_t* count_host);

/* out = sign(x) max(|x| - delta, 0), elementwise (shrink, rpca.py:99-104);
 * CORUTV_ERR_NONFINITE if x holds a non-finite entry (as_matrix,
 * dense.py:48-49).  x, out: m x n device (ld ldx / ldo; out may be x). */
int corutv_shrink(corutv_handle* h, const double* x, int64_t m, int64_t n, int64_t ldx, double delta,
                  double* out, int64_t ldo);

/* sum of squares of an m x n matrix (rpca.py:187, dense.py:94-96); in the
 * row-sharded mode the sum over all ranks.  CORUTV_ERR_NONFINITE on every
 * rank when any rank's block holds a non-finite entry. */
int corutv_sumsq(corutv_handle* h, const double* a, int64_t m, int64_t n, int64_t lda,
                 double* out_host);

/* |A - U T V'|_F without materialising U T V' — sketch.py:211-217 (K11). */
int corutv_lowrank_error(corutv_handle* h, const double* a, int64_t m, int64_t n, int64_t lda,
                         const double* u, const double* t, const double* v, int ell,
                         double* out_host);

/* Dense FP64 tensor-core GEMM primitives (the sketch contractions):
 *   trans_a == 0 : C(M x N) = A(M x K) B(K x N)          — sketch.py:149
 *   trans_a == 1 : C(M x N) = A(K x M)' B(K x N)         — sketch.py:153
 * B is K x N (ld ldb).  C has leading dimension ldc. */
int corutv_gemm(corutv_handle* h, int trans_a, int64_t M, int64_t N, int64_t K, const double* a,
                int64_t lda, const double* b, int64_t ldb, double* c, int64_t ldc);

/* Measurement hooks (bench.py): begin() resets the kernel-launch counter and
 * starts recording CUDA events on the handle's stream around every DMMA GEMM
 * and fused low-rank launch; end() synchronises and returns, per class
 * c in {0 unused, 1 = GEMMs sweeping the data matrix (K1/K2/K5), 2 = other
 * GEMMs (QR Grams / triangular products / lift), 3 = fused low-rank (ALM)}:
 * out12[3c] = summed kernel ms, out12[3c+1] = launches, out12[3c+2] =
 * algorithmic flops (2MNK); *launches = all kernels launched since begin(). */
int corutv_profile_begin(corutv_handle* h);
int corutv_profile_end(corutv_handle* h, double* out12, int64_t* launches);

#ifdef __cplusplus
}
#endif

#endif /* CORUTV_B200_H */

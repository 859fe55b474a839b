/*
 * fase_b200.h -- C ABI of the B200-native FaSE hot path (libfase_b200.so).
 *
 * The reference (`/root/reference/pkg/src/fase`) is a pure-Python package with
 * no FFI layer; its boundary is the Python API re-exported from
 * `pkg/src/fase/__init__.py:14-132`. These entry points are what a ctypes /
 * cffi binding of that API binds (INTEGRATION.md shows the stub); each one
 * names the reference function it replaces.
 *
 * Conventions
 *   - Every pointer is DEVICE memory owned by the caller (e.g. a torch tensor);
 *     the library never allocates or frees on these paths.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Work is enqueued asynchronously; errors of the enqueue are returned.
 *   - Matrices are row-major float64 with an explicit leading dimension
 *     (elements). Operands read with 16-byte vector loads require an even
 *     leading dimension and 16-byte-aligned base pointers.
 *   - Return value: FASE_OK (0) or a negative status. Status codes map 1:1 to
 *     the reference exception classes (`pkg/src/fase/errors.py:8-47`);
 *     fase_last_error() gives a thread-local message for the last failure.
 *   - No global mutable state besides that message: calls are reentrant per
 *     stream; the caller selects the device (cudaSetDevice / torch.cuda.device).
 */
#ifndef FASE_B200_H
#define FASE_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define FASE_API __attribute__((visibility("default")))
#else
#define FASE_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum {
  FASE_OK = 0,
  FASE_ERR_SHAPE = -1,          /* ShapeError            errors.py:8  */
  FASE_ERR_PARAMETER = -2,      /* ParameterError        errors.py:12 */
  FASE_ERR_MASK = -3,           /* MaskError             errors.py:16 */
  FASE_ERR_FORMAT = -4,         /* FormatError           errors.py:20 */
  FASE_ERR_DEGENERATE = -5,     /* DegenerateAtomError   errors.py:24 */
  FASE_ERR_NO_SELECTABLE = -6,  /* NoSelectableAtomError errors.py:37 */
  FASE_ERR_STALE = -7,          /* StaleTableError       errors.py:41 */
  FASE_ERR_UNSUPPORTED = -8,    /* UnsupportedDictionaryError errors.py:45 */
  FASE_ERR_CUDA = -100          /* CUDA launch / runtime failure */
};

/* Thread-local text of the last non-OK status of this thread. */
FASE_API const char* fase_last_error(void);

/* ABI version: (major << 16) | minor. */
FASE_API int fase_abi_version(void);

/* Largest dictionary size K fase_iterate accepts (real tables). Up to
 * fase_iterate_register_atoms() the recursion keeps R in registers; beyond it a
 * streaming recursion (csrc/iterate_generic.cu, bit-identical arithmetic) keeps
 * R in the caller's R_out, which is then required (it may alias R0; no R_log),
 * and the scaled / fused-synthesis entry points are not available. */
FASE_API int fase_max_atoms(void);
FASE_API int fase_iterate_register_atoms(void);

/* Leading dimension (>= K, even) that table rows handed to fase_iterate must
 * have, zero-padded past K; 0 if K is unsupported. */
FASE_API int fase_table_ld(int K);

/*
 * Basis construction (replaces the separable branch of generate_dictionary,
 * dictionary.py:167-178, np.einsum("um,vn->uvmn")):
 *   phi[(row0 + u*Lc + v) * ldphi + m*Nc + n] = rows[u*Mr + m] * cols[v*Nc + n]
 * one correctly rounded multiply per sample, bit-identical to the einsum.
 */
FASE_API int fase_basis_outer(const double* rows, int Lr, int Mr, const double* cols, int Lc, int Nc,
                     double* phi, int64_t ldphi, int64_t row0, void* stream);

/*
 * Weighted Gram table (replaces build_gram_tables, fast.py:109-142):
 *   G[k*ldg + l] = sum_m (phi[k,m] * w[m]) * phi[l,m]      for k, l < K, m < M
 * Phi o w is formed in `ws` (fase_gram_workspace(K, M) bytes, 16-byte aligned),
 * then FP64 DMMA tiles compute the upper triangle and mirror it exactly, so G
 * is bit-symmetric.
 */
FASE_API size_t fase_gram_workspace(int K, int M);
FASE_API int fase_gram(const double* phi, int64_t ldphi, const double* w, int K, int M,
                       double* G, int64_t ldg, void* ws, size_t ws_bytes, void* stream);

/*
 * Plain FP64 contraction C[i*ldc + j] = sum_k A[i*lda + k] * B[j*ldb + k]
 * (the DMMA tile kernel behind fase_gram / fase_init_products; variant 0 is
 * the library's tile, 1 an alternative tile kept for measurement).
 */
FASE_API int fase_gemm_nt(const double* A, int64_t lda, const double* B, int64_t ldb, int M,
                          int N, int Kd, double* C, int64_t ldc, int variant, void* stream);

/*
 * Normalizers (replaces _finish_tables, fast.py:97-106):
 *   top = max_k G[k,k];  D[k] = (top > 0 && G[k,k] > 1e-12*top) ? 1/sqrt(G[k,k]) : 0
 * `n_alive` (device int32, may be NULL) receives the number of non-degenerate atoms.
 */
FASE_API int fase_gram_finish(const double* G, int64_t ldg, int K, double* D, int32_t* n_alive,
                     void* stream);

/*
 * Batched initial scalar products (replaces initial_scalar_products,
 * fast.py:145-157, one zgemv per block):
 *   R0[b*ldr + k] = sum_m (f[b*ldf + m] * w[b*ldw + m]) * phi[k*ldphi + m]
 * ldw == 0 shares one weight vector across the batch. F o W is formed in `ws`
 * (fase_init_products_workspace(M, B) bytes), then one DMMA GEMM.
 */
FASE_API size_t fase_init_products_workspace(int M, int B);
FASE_API int fase_init_products(const double* phi, int64_t ldphi, const double* f, int64_t ldf,
                                const double* w, int64_t ldw, int K, int M, int B,
                                double* R0, int64_t ldr, void* ws, size_t ws_bytes,
                                void* stream);

/*
 * Weighted operand: out[b*ldo + m] = x[b*ldx + m] * w[b*ldw + m] (ldw == 0:
 * one shared weight row), one correctly rounded multiply per sample -- the
 * reference's `s * w` (fast.py:154). Even leading dimensions.
 */
FASE_API int fase_weigh(const double* x, int64_t ldx, const double* w, int64_t ldw, int rows,
                        int M, double* out, int64_t ldo, void* stream);

/*
 * Weighted operand on the samples with nonzero weight (the support):
 *   out[b*ldo + i] = x[b*ldx + idx[i]] * w[i]   for i < n, zero-padded to even n
 * With Phi's columns gathered the same way once, fase_gemm_nt over n instead of
 * M samples gives the same products: lost samples add exact zeros
 * (initial_scalar_products, fast.py:154, over the support only).
 */
FASE_API int fase_weigh_gather(const double* x, int64_t ldx, const int32_t* idx, const double* w,
                               int rows, int n, double* out, int64_t ldo, void* stream);

/*
 * Initial products of one separable dictionary part (atoms
 * phi[col0 + u*Lc + v](m, n) = rows[u, m] * cols[v, n], dictionary.py:167-178)
 * for B weighted areas X (B x ldx, Mr*Nc samples each, e.g. the F o W formed
 * by fase_init_products' first step or by fase_frame_areas):
 *   R0[b*ldr + col0 + u*Lc + v] = (rows X_b cols^T)[u, v]
 * -- the separable-transform form of initial_scalar_products (fast.py:145-157),
 * 2(Lr*Mr*Nc + Lr*Nc*Lc) flops per block instead of 2*Lr*Lc*Mr*Nc.
 */
FASE_API int fase_sep_products(const double* rows, int Lr, int Mr, const double* cols, int Lc,
                               int Nc, const double* X, int64_t ldx, int B, double* R0,
                               int64_t ldr, int64_t col0, void* stream);

/*
 * All separable parts of a dictionary at once on the FP64 tensor cores
 * (mma.sync f64), with the weights applied while staging the area:
 *   X_b = F_b o W (W == NULL: F is already weighted; ldw == 0: one shared W)
 *   R0[b*ldr + col0_p + u*Lc_p + v] = (rows_p X_b cols_p^T)[u, v]   for every part p
 * -- fase_weigh + fase_sep_products for up to 8 parts in one launch.
 */
typedef struct {
  const double* rows; /* Lr x Mr */
  int Lr;
  const double* cols; /* Lc x Nc */
  int Lc;
  int64_t col0;
} fase_sep_part;

FASE_API int fase_sep_products_batch(const fase_sep_part* parts, int n_parts, int Mr, int Nc,
                                     const double* F, int64_t ldf, const double* W, int64_t ldw,
                                     int B, double* R0, int64_t ldr, void* stream);

/*
 * Per-block normalizers for per-block geometries whose table rows are
 * G_b = G0 - sum_{j in chunks(b)} C_j (see fase_iterate):
 *   diag_b[k] = G0[k,k] - sum_j C_j[k,k];  D[b*ldd + k] as in fase_gram_finish.
 * n_alive[b] receives the count of non-degenerate atoms of block b.
 * ldg == 0: G0 and the chunk tables are passed as their diagonals instead
 * (G0[k] and chunk_tables[j*chunk_stride + k]); same values, same order.
 */
FASE_API int fase_block_normalizers(const double* G0, int64_t ldg, const double* chunk_tables,
                           int64_t chunk_stride, const int32_t* chunk_count,
                           const int32_t* chunk_ids, int64_t chunk_list_ld, int K, int B,
                           double* D, int64_t ldd, int32_t* n_alive, void* stream);

/*
 * The FaSE recursion for B independent blocks (replaces the loop of
 * fase_extrapolate, fast.py:224-255, with the tie rule of reference.py:55-85):
 *   metric_k = |R_k| * D_k  (D_k == 0: never selectable)
 *   q = max(q, 1e-13 * max metric);  u = lowest k with metric_k >= max - q
 *   p = R_u * (D_u * D_u);  c = gamma * p;  R_k <- R_k - c * row_u[k]
 * row_u = G0[u, :] - sum_{j in chunks(b)} C_j[u, :]   (no chunk lists when
 * chunk_count == NULL: shared geometry). One persistent CTA per block keeps R and
 * D in registers; rows are streamed with 16-byte loads. G0 / C_j rows must be
 * zero-padded to ldg >= fase_table_ld(K).
 *   R0, R_out: B x ldr (R_out may be NULL or alias R0)
 *   D: shared vector (ldd == 0) or B x ldd
 *   sel / proj / coef: B x ldo outputs (I entries per block)
 *   R_log: NULL or B x I x ldr record of R after every iteration
 * Precomposed bases (optional, chunked geometries): compose != NULL is an
 * n_compose^compose_depth table (compose_depth 1..3) indexed by a list prefix
 * padded with its last entry, e.g. depth 3: (c1, c2, c3), (c1, c2, c2), (c1, c1, c1).
 * For the longest prefix of length k <= compose_depth of a block's (ascending)
 * list with p = compose[prefix] > 0:
 *   row_u = B_p[u, :] - sum over the list's remaining chunks,
 * B_p = G0 + p * base_stride, which must hold G0 - C_c1 - ... - C_ck composed
 * element by element in list order (so the rows are bit-identical to the
 * uncomposed ones). Normalizers are unaffected (fase_block_normalizers takes
 * the full lists).
 */
typedef struct {
  const double* G0;
  int64_t ldg;
  const double* chunk_tables; /* C_j = chunk_tables + j * chunk_stride, row stride ldg */
  int64_t chunk_stride;
  const int32_t* chunk_count; /* B list lengths, or NULL: shared geometry */
  const int32_t* chunk_ids;   /* B x chunk_list_ld table ids, each list in order */
  int64_t chunk_list_ld;
  const double* D;
  int64_t ldd;
  const double* R0;
  int64_t ldr;
  double* R_out;
  double* R_log;
  int K;
  int B;
  int I;
  double gamma;
  int32_t* sel;
  double* proj;
  double* coef;
  int64_t ldo;
  const int32_t* compose; /* NULL, or n_compose^compose_depth base indices (see above) */
  int n_compose;
  int compose_depth;
  int64_t base_stride;
  /* optional L2 residency hint (shared geometries): bit u of l2_hot[u / 32] set
   * = row u is "hot" (frequently selected): its staged-row copies carry an
   * L2 evict_last policy, every other row evict_first, so the hot rows stay
   * L2-resident. NULL: default policy. Does not change any result. */
  const uint32_t* l2_hot;
  /* optional dispatch order (ABI 3.0): NULL, or a permutation of 0..B-1, and
   * the i-th CTA (slot) runs block order[i]. Blocks are independent, so only the
   * schedule changes, never a result: per-block geometries put their costliest
   * blocks first (fase_block_order) so the last wave holds the cheap ones. Only
   * the chunk-list recursions (and the streaming one) honour it: shared
   * geometries, whose blocks cost the same, run slot order. */
  const int32_t* order;
} fase_iterate_args;

FASE_API int fase_iterate(const fase_iterate_args* args, void* stream);

/*
 * Scaled recursion for shared geometries (same loop as fase_iterate, fast.py:
 * 238-255, in scaled variables): G0 is the column-scaled table
 *   Gs[u, k] = G[u, k] * D_k            (fase_scale_columns)
 * and the kernel carries R'_k = R_k * D_k, so the metric is |R'_k| and the
 * update R' -= c * Gs[u, :] needs no normalizers; p = R'_u * D_u, c = gamma*p.
 * R0 and D are the unscaled inputs of fase_iterate (D shared, ldd = 0).
 * Iteration 0 is bit-identical to fase_iterate; later iterations differ by the
 * rounding of the scaled operands, so a selection can differ only where the
 * top-two metrics lie within a few ulp (the north-star tolerance: top-two
 * within 1e-9 relative; coefficients within 1e-6). chunk lists, compose,
 * per-block D, R_out and R_log are rejected (FASE_ERR_UNSUPPORTED).
 */
typedef struct {
  const double* phi; /* K x ldphi: the atoms restricted to the lost samples (16-byte aligned) */
  int64_t ldphi;     /* even, >= n_lost */
  int n_lost;
  double* out;       /* out[b*ldout + i] = g_i of block b (packed lost samples) */
  int64_t ldout;
} fase_synth_fused;

/* synth == NULL: recursion only. Otherwise the synthesis of fase_synth_paste
 * (packed output, dst = 0..n_lost-1) is fused into the recursion: each
 * iteration adds c * phi[u, i] in selection order, bit-identical to a
 * separate fase_synth_paste over the same terms. n_lost must not exceed
 * fase_iterate_scaled_synth_capacity(K, B) (else FASE_ERR_UNSUPPORTED). */
FASE_API int fase_iterate_scaled(const fase_iterate_args* args, const fase_synth_fused* synth,
                                 void* stream);
FASE_API int fase_iterate_scaled_synth_capacity(int K, int B);

/* The exact recursion (fase_iterate, bit-identical selections / coefficients)
 * with the synthesis fused in, for shared geometries and batches of at most one
 * block per SM (latency-bound: config 0): bit-identical to fase_iterate
 * followed by fase_synth_paste over the packed lost samples. n_lost must not
 * exceed fase_iterate_synth_capacity(K, B) (0: not available for this batch). */
FASE_API int fase_iterate_synth(const fase_iterate_args* args, const fase_synth_fused* synth,
                                void* stream);
FASE_API int fase_iterate_synth_capacity(int K, int B);

/* Gs[u*lds + k] = G[u*ldg + k] * D[k] (u < rows, k < K), 0 for K <= k < lds;
 * lds even. A complex table (rows of conj(C)) is scaled as its real view:
 * rows = K, 2K columns, D repeated per (re, im) pair. */
FASE_API int fase_scale_columns(const double* G, int64_t ldg, const double* D, int rows, int K,
                                double* Gs, int64_t lds, void* stream);

/*
 * Model synthesis and paste (replaces SparseModel.materialize + apply_model,
 * reference.py:120-125 and fast.py:267-286, evaluated on lost samples only):
 *   g = sum_t coef[b,t] * phi[sel[b,t], m]   accumulated in selection order
 * For output position i of block b (list position i' = idx_ptr[b] + i, or
 * i' = i for one shared list of n_shared samples when idx_ptr == NULL; the
 * area sample is m = idx[i']):
 *   dst == NULL : out[b*ldout + m]        = g   (patch (B, ldout) areas in place)
 *   dst != NULL : out[b*ldout + dst[i']]  = g   (ldout = 0: paste into a frame at
 *                                                absolute offsets; dst = 0..n-1 with
 *                                                ldout = n: packed lost samples)
 */
FASE_API int fase_synth_paste(const double* phi, int64_t ldphi, const int32_t* sel, const double* coef,
                     int64_t ldo, int I, int B, const int32_t* idx_ptr, const int32_t* idx,
                     int n_shared, const int64_t* dst, double* out, int64_t ldout, void* stream);

/*
 * Frame concealment (replaces the per-tile body of conceal_image,
 * conceal.py:111-148, for every lossy tile of a frame at once). Losses are
 * whole tiles: grid is the (H/tile) x (W/tile) tile loss map (nonzero = lost);
 * corners (L x 2, int32) are the top-left pixels of the lossy tiles; areas are
 * A x A with A = tile + 2*support, out-of-frame samples unavailable.
 *
 * fase_frame_areas: X[b, i*A + j] = frame(r0-s+i, c0-s+j) * base_w[i*A + j] on
 *   support samples, 0 elsewhere -- the weighted operand of the initial products.
 * fase_frame_cells: counts[b], ids[b, :] = the candidate cells (rectangles of
 *   the area, one representative sample (i, j) each in cell_rep) unavailable
 *   for block b -- the chunk lists of fase_iterate / fase_block_normalizers.
 * fase_frame_paste: the tile's own lost pixels <- sum_t coef * phi[sel, m]
 *   (conceal.py:144-148).
 */
FASE_API int fase_frame_areas(const double* frame, int64_t ldf, const uint8_t* grid,
                              int64_t ldgrid, int H, int W, int tile, int support,
                              const int32_t* corners, int L, const double* base_w, double* X,
                              int64_t ldx, void* stream);
FASE_API int fase_frame_cells(const uint8_t* grid, int64_t ldgrid, int H, int W, int tile,
                              int support, const int32_t* corners, int L,
                              const int32_t* cell_rep, int n_cells, int32_t* counts,
                              int32_t* ids, int64_t ids_ld, void* stream);
/* fase_block_order: order = the blocks 0..B-1 by descending cost class
 * min(7, max(0, counts[b] - depth)) -- the chunk-table rows a block streams per
 * iteration beyond its (precomposed) base when compose_depth = depth -- stable
 * (ascending block index within a class); the fase_iterate_args.order of the
 * frame's recursion (longest-processing-time-first dispatch). */
FASE_API int fase_block_order(const int32_t* counts, int B, int depth, int32_t* order,
                              void* stream);
FASE_API int fase_frame_paste(const double* phi, int64_t ldphi, const int32_t* sel,
                              const double* coef, int64_t ldo, int I, const uint8_t* grid,
                              int64_t ldgrid, int H, int W, int tile, int support,
                              const int32_t* corners, int L, double* out, int64_t ldout,
                              void* stream);
/* fase_frame_paste for complex dictionaries: phi2 in the conjugate-split
 * layout (rows 2u = Re phi_u, 2u+1 = -Im phi_u), coef interleaved complex (ldo
 * in complex elements); Re g is pasted and, when max_imag != NULL,
 * max_imag[b] = max |Im g| over tile b's pixels (apply_model, fast.py:267-286). */
FASE_API int fase_frame_paste_complex(const double* phi2, int64_t ldphi, const int32_t* sel,
                                      const double* coef, int64_t ldo, int I, const uint8_t* grid,
                                      int64_t ldgrid, int H, int W, int tile, int support,
                                      const int32_t* corners, int L, double* out, int64_t ldout,
                                      double* max_imag, void* stream);
/*
 * fase_frame_widen: out[y, x] = lost[y, x] ? 0.0 : (double)frame_u8[y, x] -- the
 * damaged float64 frame the pipeline conceals, from the uint8 luma the caller
 * uploads (pgm.py / conceal_image's `observed` with lost pixels zeroed,
 * conceal.py:167-200). lost: H x W bytes, nonzero = lost.
 */
FASE_API int fase_frame_widen(const uint8_t* frame_u8, int64_t ldu, const uint8_t* lost,
                              int64_t ldl, int H, int W, double* out, int64_t ldout,
                              void* stream);

/*
 * ---- Complex-valued dictionaries (dft, bdft, their unions; dictionary.py:126-166)
 *
 * Device layout of a complex dictionary ("conjugate-split"): 2K rows of ldphi
 * doubles, row 2k = Re phi_k, row 2k+1 = -Im phi_k. Passed to
 * fase_init_products as a real dictionary of 2K atoms it yields
 * conj(Phi) (F o W) interleaved -- R0[b, k] = (re, im) -- which is
 * initial_scalar_products' conj(phi @ conj(s*w)) (fast.py:154-155).
 *
 * Complex tables are rows of interleaved (re, im) doubles; ldt counts complex
 * elements. The table stores conj(C[u, :]) -- the operand of the update
 * (fast.py:246) -- exactly Hermitian with a real diagonal:
 *   T[u*ldt + l] = conj(C[u, l]),  C = conj(Phi) W Phi^T   (fast.py:109-142)
 * Normalizers of a complex table come from fase_gram_finish(T, 2*ldt + 1, ...)
 * (the real parts of the diagonal sit at stride 2*ldt + 2 doubles); per-block
 * chunked normalizers likewise pass ldg = 2*ldt + 1 and a stride in doubles.
 */
FASE_API size_t fase_gram_complex_workspace(int K, int64_t ldphi);
FASE_API int fase_gram_complex(const double* phi2, int64_t ldphi, const double* w, int K, int M,
                               double* T, int64_t ldt, void* ws, size_t ws_bytes, void* stream);

/* Largest K / table leading dimension (complex elements) of fase_iterate_complex. */
FASE_API int fase_max_atoms_complex(void);
FASE_API int fase_table_ld_complex(int K);
/* Largest complex K whose recursion keeps R in registers; beyond it (up to
 * fase_max_atoms_complex()) fase_iterate_complex runs the streaming recursion
 * (csrc/iterate_generic.cu, same arithmetic), which needs R_out (may alias R0). */
FASE_API int fase_iterate_complex_register_atoms(void);

/*
 * The recursion in complex128 (fast.py:224-255): metric |R_k| * D_k with numpy's
 * complex abs, the same tie rule, p = R_u * (D_u * D_u), c = gamma * p and
 * R_k <- R_k - c * T[u, k] with numpy's complex product; bit-identical to the
 * reference given the same R0 / table / D. Same argument block as fase_iterate
 * with these units: G0 / chunk tables are complex tables (ldg, chunk_stride in
 * complex elements, ldg >= fase_table_ld_complex(K)); R0 / R_out / R_log
 * interleaved complex with ldr in complex elements; proj / coef interleaved
 * complex (B x ldo complex); D, sel as in fase_iterate.
 */
FASE_API int fase_iterate_complex(const fase_iterate_args* args, void* stream);

/* The scaled recursion for complex dictionaries (see fase_iterate_scaled):
 * G0 holds column-scaled rows conj(C)[u, k] * D_k (fase_scale_columns on the
 * real view), R' = R * D, the metric |R'|; shared geometry only. */
FASE_API int fase_iterate_complex_scaled(const fase_iterate_args* args, void* stream);

/*
 * Complex model synthesis and paste (SparseModel.materialize + apply_model):
 * as fase_synth_paste with phi2 in the conjugate-split layout and coef
 * interleaved complex; Re g is written to out and, when max_imag != NULL,
 * max_imag[b] = max |Im g| over block b's samples (apply_model's second result,
 * fast.py:284).
 */
FASE_API int fase_synth_paste_complex(const double* phi2, int64_t ldphi, const int32_t* sel,
                                      const double* coef, int64_t ldo, int I, int B,
                                      const int32_t* idx_ptr, const int32_t* idx, int n_shared,
                                      const int64_t* dst, double* out, int64_t ldout,
                                      double* max_imag, void* stream);

/*
 * Transform shortcuts (transform.py:43-110).
 *
 * fase_sep_products_complex: initial products of one complex separable part,
 * atoms phi[col0 + u*Lc + v](m, n) = E[u, m] * F[v, n] (E = rows_re + i rows_im,
 * F = cols_re + i cols_im; the DFT exponentials of dictionary.py:126-131), for
 * B real weighted areas X:
 *   R0[b*ldr + col0 + u*Lc + v] = sum_{m,n} conj(E[u,m]) conj(F[v,n]) X_b[m,n]
 * (R0 interleaved complex, ldr in complex elements). For the full exponential
 * grid this is fft2(X_b) -- fft_initial_products' identity -- at
 * 2 (2 Lc Mr Nc + 4 Lr Lc Mr) flops per block instead of 4 Lr Lc Mr Nc.
 *
 * fase_fft_gram: the complex table of a frequency-tagged dictionary from the
 * spectrum of its weight, spec = fft2(w) (M*N interleaved complex, e.g. from
 * fase_sep_products_complex with X = w): S = (spec + conj(spec[-a,-b])) / 2,
 *   T[k*ldt + l] = conj(C(k, l)) = S[(mu_l - mu_k) mod M, (eta_l - eta_k) mod N]
 * zero-padded past K, exactly Hermitian with a real diagonal (fft_gram_table,
 * transform.py:84-110). mu / eta: K int32 tags, or both NULL for the canonical
 * order k = mu*N + eta.
 */
FASE_API int fase_sep_products_complex(const double* rows_re, const double* rows_im, int Lr, int Mr,
                                       const double* cols_re, const double* cols_im, int Lc, int Nc,
                                       const double* X, int64_t ldx, int B, double* R0, int64_t ldr,
                                       int64_t col0, void* stream);
FASE_API int fase_fft_gram(const double* spec, int M, int N, const int32_t* mu, const int32_t* eta,
                           int K, double* T, int64_t ldt, void* stream);

/*
 * FP64 contractions on the tcgen05 tensor cores (Ozaki scheme, kind::i8):
 *
 * fase_ozaki_split: digit planes of `rows` FP64 rows of length kd, with
 * v[r,k] = x[r*ldx + (idx ? idx[k] : k)] * (w ? w[k] : 1) (one rounding: the
 * support-restricted weighted operand of fase_weigh_gather, or x itself):
 *   e[r] = min e with max_k |v[r,k]| < 2^e;
 *   v[r,k] = 2^e[r] * sum_{i<slices} digit_i[r,k] * 2^{-7(i+1)} + residual
 * (signed 7-bit digits, truncated; kd zero-padded to kp, a multiple of 64;
 * slices 6..8).
 * Plane i occupies rows_pad * kp bytes at planes + i * rows_pad * kp, stored
 * in the UMMA-ready tiled order [k / 64][r / 8][(k / 16) % 4][r % 8][k % 16].
 *
 * fase_ozaki_gemm: C[r*ldc + c] = sum_k X[r,k] Y[c,k] from the planes of X
 * (a_rows_pad a multiple of 128) and Y (b_rows_pad a multiple of 64): int8 x
 * int8 -> int32 tcgen05 MMAs for every digit pair i + j <= slices - 1
 * (0-based), one TMEM accumulator per diagonal, combined in FP64 and scaled by
 * 2^(e_X[r] + e_Y[c]). With 8 planes the result matches an FP64 contraction
 * to rounding level (initial_scalar_products, fast.py:145-157, on the support).
 */
FASE_API int fase_ozaki_split(const double* x, int64_t ldx, const int32_t* idx, const double* w,
                              int rows, int kd, int slices, int8_t* planes, int64_t kp,
                              int rows_pad, int32_t* exps, void* stream);
FASE_API int fase_ozaki_gemm(const int8_t* a_planes, int a_rows_pad, const int32_t* ea,
                             int m_rows, const int8_t* b_planes, int b_rows_pad,
                             const int32_t* eb, int n_rows, int64_t kp, int slices, double* C,
                             int64_t ldc, void* stream);
/* Synthesis of a shared geometry's lost samples as one Ozaki product
 * (SparseModel.materialize, reference.py:120-125, at the lost samples; the
 * plan's batched apply_model, fast.py:267-286): row r of V is block r's sparse
 * model scattered to a dense coefficient vector, v[r, sel[r*ldsel + t]] +=
 * coef[r*ldcoef + t] for t < iters (sel < 0 or >= kd: no term; repeated atoms
 * summed in term order), cut into digit planes exactly like
 * fase_ozaki_split; then fase_ozaki_gemm(V planes, Phi_lost^T planes) gives
 * g[r, i] = sum_k v[r, k] phi_k[lost_i] to the planes' precision. */
FASE_API int fase_ozaki_split_sparse(const int32_t* sel, int64_t ldsel, const double* coef,
                                     int64_t ldcoef, int rows, int iters, int kd, int slices,
                                     int8_t* planes, int64_t kp, int rows_pad, int32_t* exps,
                                     void* stream);
/* The weighted Gram table on the same path (build_gram_tables, fast.py:109-142):
 * planes of Phi o w (A) and Phi (B), K rows each; only tiles holding entries
 * k <= l are computed, each such entry written to (k, l) and (l, k): G is
 * bit-symmetric, like fase_gram's. */
FASE_API int fase_ozaki_gram(const int8_t* a_planes, int a_rows_pad, const int32_t* ea,
                             const int8_t* b_planes, int b_rows_pad, const int32_t* eb, int K,
                             int64_t kp, int slices, double* G, int64_t ldg, void* stream);

/* Writes `bytes` of zeros-then-ones into `buf` to evict L2 between timed steps. */
/* G[i*ldg + j] <- G[j*ldg + i] for K > i > j: a table assembled from row
 * panels (multi-GPU build, each rank's rows of the non-symmetric product)
 * becomes the exact mirror of its upper triangle, bit-identical to the
 * single-GPU symmetric build (fase_gram / fase_ozaki_gram write that mirror). */
FASE_API int fase_mirror_upper(double* G, int64_t ldg, int K, void* stream);
FASE_API int fase_l2_flush(void* buf, size_t bytes, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* FASE_B200_H */

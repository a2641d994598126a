/*
 * fdp.h -- C ABI of the B200-native Fast-Diagonalization block preconditioner
 * (M. Montardini, G. Sangalli, M. Tani, "Robust isogeometric preconditioners for the Stokes
 * system based on the Fast Diagonalization method", arXiv:1712.00403).
 *
 * Citations "P:L" are lines of the paper text with the section / equation named.
 *
 * Conventions for every entry point
 *   - Plain C99 types only. Matrices on the host are dense, column-major, n x n.
 *   - Tensors are vectors in vec order, i1 fastest: i = i1 + n1*(i2 + n2*i3) (§2.3).
 *     A batch of B vectors is stored batch-major: item b starts at offset b*N.
 *   - "device" pointers are CUDA global-memory pointers on the handle's device; passing a host
 *     pointer where a device pointer is required returns FDP_ERR_INVALID_ARG.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream). Apply calls are
 *     asynchronous on that stream, allocate nothing and never synchronise (except the *_host
 *     variant), so they are CUDA-graph capturable. Launch failures return FDP_ERR_CUDA; faults
 *     during execution surface at the caller's next synchronisation.
 *   - Handles own their device memory; caller arrays are copied at setup. Destroy after the
 *     caller has synchronised every stream that used the handle. Destroy functions are NULL-safe.
 *   - No function aborts, exits or throws across the ABI. On failure the status is returned and
 *     fdp_last_error() (thread-local) holds a one-line message.
 *   - There is no CPU fallback: every apply runs in this library's sm_100a kernels.
 */
#ifndef FDP_H_
#define FDP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FDP_OK = 0,
  FDP_ERR_INVALID_ARG = 1, /* null / host-vs-device pointer mix-up / bad enum */
  FDP_ERR_SHAPE = 2,       /* dimension out of range or inconsistent */
  FDP_ERR_NOT_SPD = 3,     /* Cholesky of a mass matrix failed, or matrix not symmetric */
  FDP_ERR_SINGULAR = 4,    /* Kronecker-sum spectrum: sum_d c_d min(lambda_d) <= 1e-12 sum_d c_d max(lambda_d) */
  FDP_ERR_CUDA = 5,        /* CUDA runtime error (launch, copy, graph) */
  FDP_ERR_OOM = 6,         /* device or host allocation failed */
  FDP_ERR_NCCL = 7,        /* NCCL unavailable (libnccl.so.2 not loadable) or an NCCL call failed */
  FDP_ERR_UNSUPPORTED = 8  /* valid request this build does not implement (e.g. D > 3) */
} fdp_status;

const char* fdp_status_string(fdp_status s);
/* Thread-local message of the last failing call on this thread ("" if none). */
const char* fdp_last_error(void);
/* Library version string, e.g. "fdp 0.1 sm_100a". */
const char* fdp_version(void);

/* ------------------------------------------------------------------------------------------
 * Host helpers: univariate isogeometric factors ("univariate matrix factors", §5;
 * P:734-737 pressure mass). Built by this library's own B-spline evaluation and Gauss rule.
 * ------------------------------------------------------------------------------------------ */
enum {
  FDP_IGA_INTERIOR = 1, /* restrict to basis functions l,s = 2..m-1 (Dirichlet / normal trace,
                           P:265-267, 694, 699) */
  FDP_IGA_NITSCHE = 2   /* replace K by K~ of P:701-704 (tangential RT factor, Nitsche bracket
                           with penalty 2*c_pen/h, h = 1/n_el) */
};

/* Open uniform knot vector of degree `deg`, uniform regularity `alpha` (-1 <= alpha < deg),
 * n_el elements. Writes K (stiffness, int b_l' b_s') and M (mass, int b_l b_s) as
 * column-major n x n into caller-owned host arrays of at least n*n doubles, where n is the
 * space dimension m = n_el(deg-alpha)+alpha+1, minus 2 with FDP_IGA_INTERIOR. Gauss rule with
 * `q` points per element (q <= 0 selects deg+1, exact for these polynomial integrands).
 * K or M may be NULL to skip it; both NULL just reports n in *n_out.
 * Errors: FDP_ERR_SHAPE (deg < 1, alpha out of range, n_el < 1, n < 1), FDP_ERR_INVALID_ARG. */
fdp_status iga_univariate(int deg, int alpha, int n_el, int flags, double c_pen, int q,
                          double* K, double* M, int32_t* n_out);

/* Greville abscissae (xi_{j+1}+...+xi_{j+deg})/deg of the same space (first/last dropped with
 * FDP_IGA_INTERIOR): dof coordinates used to sample a coefficient at dofs (C-6).
 * g: host array of at least n doubles, or NULL to query n. */
fdp_status iga_greville(int deg, int alpha, int n_el, int flags, double* g, int32_t* n_out);

/* Diagonal scaling sampled at dofs from a coefficient written as a sum of separable terms,
 * nu(x) = sum_t c[t] prod_d f_td(x_d) (config 3's nu = 1 + 0.5 sin(2 pi x) sin(2 pi y) sin(2 pi z),
 * DESIGN.md C-6): out[i] = v_i (invert = 0) or 1 / v_i (invert = 1), with
 * v_i = sum_t c[t] prod_d f[t*D + d][i_d], i = i_1 + n_1 (i_2 + n_2 i_3) (vec order, i1 fastest,
 * P:382-386). f[t*D + d]: host array of n[d] values of the factor at the direction-d dof points
 * (e.g. iga_greville), or NULL for a factor identically 1. D in [1, 3], T >= 1; out: host array
 * of prod n[d] doubles. Errors: FDP_ERR_SHAPE (D, T or n out of range), FDP_ERR_INVALID_ARG
 * (NULL out / n / c / f, or a zero sum with invert = 1). */
fdp_status fdp_kron_diag(int D, const int32_t* n, int T, const double* const* f, const double* c,
                         int invert, double* out);

/* Generalized symmetric-definite eigenproblem K U = M U diag(lambda), U^T M U = I (Algorithm 1
 * step 1), host only: the routine fd_setup uses. K, M: host column-major n x n, M SPD;
 * U (n*n, column j = eigenvector j, largest-magnitude entry positive) and lambda (n, ascending)
 * are caller-owned host arrays. Errors: FDP_ERR_SHAPE, FDP_ERR_NOT_SPD, FDP_ERR_SINGULAR (QL
 * iteration did not converge). */
fdp_status fdp_gen_eig(int n, const double* K, const double* M, double* U, double* lambda);

/* ------------------------------------------------------------------------------------------
 * FD solver for one Sylvester-like Kronecker system (Algorithm 1, §5.2):
 *   R = sum_d coef[d] * (F_D (x) ... (x) F_1),  F_e = K_e if e == d else M_e
 *   x = dscale o ( U Lambda^{-1} U^T ( dscale o b ) ),  U = U_D (x) ... (x) U_1,
 *   Lambda = sum_d coef[d] lambda_d,  K_d U_d = M_d U_d diag(lambda_d),  U_d^T M_d U_d = I.
 * dscale = D^{-1/2} realises P^G = D^{1/2} P D^{1/2} (§6).
 * ------------------------------------------------------------------------------------------ */
typedef struct fdp_fd_s* fdp_fd;

/* D in {2,3}; n[d] in [1, 2048]; K[d], M[d]: host, column-major n[d] x n[d], symmetric to
 * 1e-12 relative, M[d] SPD; coef[d] > 0. Performs the D generalized eigensolves on the host
 * (Algorithm 1 step 1: Cholesky + Householder tridiagonalisation + implicit QL),
 * uploads U_d, U_d^T (zero padded; for persymmetric pencils the even-odd folded blocks and
 * their TMA-fragment layout) and lambda_d to `device`, and allocates a workspace for up to
 * max_batch right-hand sides (0 = none; then fd_apply needs a caller workspace). When the last
 * mode is longer than 96 and folded, the handle also holds 1 / Lambda in the Lambda pass's
 * output layout (n1p * n2 * n3 doubles, n1p = n1 rounded up to even; C-11).
 * Errors: FDP_ERR_SHAPE, FDP_ERR_NOT_SPD, FDP_ERR_SINGULAR, FDP_ERR_OOM, FDP_ERR_CUDA. */
fdp_status fd_setup(int D, const int32_t* n, const double* const* K, const double* const* M,
                    const double* coef, int device, int64_t max_batch, fdp_fd* out);

/* Host copies of U_d (column-major n_d x n_d, column j = eigenvector j) and lambda_d
 * (ascending). Either output may be NULL. */
fdp_status fd_get_eigs(fdp_fd h, int d, double* U_out, double* lambda_out);
/* N = prod n_d of the handle. */
int64_t fd_size(fdp_fd h);
/* Bytes of device workspace fd_apply needs for `batch` right-hand sides. */
size_t fd_workspace_bytes(fdp_fd h, int64_t batch);

/* b, x: device, batch*N doubles, batch-major; x may alias b (in place). dscale: device, N
 * doubles holding D^{-1/2} (> 0), or NULL for the plain solve. workspace: device, at least
 * fd_workspace_bytes(h,batch) bytes, or NULL to use the handle's own (then batch <= max_batch
 * and the handle must not be used concurrently on two streams). */
fdp_status fd_apply(fdp_fd h, const double* b, double* x, const double* dscale, int64_t batch,
                    void* workspace, void* stream);
fdp_status fd_destroy(fdp_fd h);

/* ------------------------------------------------------------------------------------------
 * Kronecker mass P_Q = M_D (x) ... (x) M_1 (eq. precQ) and its inverse by per-mode banded
 * Cholesky solves in O(p n_Q) flops (identity (A(x)B(x)C)^{-1} vec X).
 * ------------------------------------------------------------------------------------------ */
typedef struct fdp_mass_s* fdp_mass;
enum { FDP_MASS_INVERSE = 0, FDP_MASS_FORWARD = 1 };

/* M[d]: host, column-major, symmetric positive definite, half-bandwidth <= 15 (detected).
 * Errors: FDP_ERR_SHAPE, FDP_ERR_NOT_SPD, FDP_ERR_OOM, FDP_ERR_CUDA. */
fdp_status kron_mass_setup(int D, const int32_t* n, const double* const* M, int device,
                           fdp_mass* out);
int64_t kron_mass_size(fdp_mass h);
/* mode FDP_MASS_INVERSE: x = dscale o (P_Q^{-1} (dscale o b)), dscale = D_Q^{-1/2} or NULL
 * (P_Q^G of P:1039). mode FDP_MASS_FORWARD: x = P_Q b (dscale must be NULL). b, x device,
 * batch*N doubles; x may alias b for FDP_MASS_INVERSE only. No workspace is needed. */
fdp_status kron_mass_apply(fdp_mass h, int mode, const double* b, double* x,
                           const double* dscale, int64_t batch, void* stream);
fdp_status kron_mass_destroy(fdp_mass h);

/* ------------------------------------------------------------------------------------------
 * Block-diagonal preconditioner P_D = diag(P_V,1, ..., P_V,D, P_Q) (eq. P_D; P_V
 * block diagonal P:644-652) and its scaled variant P_D^G.
 * r, s layout per batch item: [u_1 | ... | u_D | p], each block in vec order.
 * ------------------------------------------------------------------------------------------ */
typedef struct fdp_block_s* fdp_block;

/* vel[k]: FD handles of the D velocity components (non-owning; must outlive the block);
 * pres: mass handle (non-owning). dscale_vel: host, sum_k N_k doubles of D_V (> 0), or NULL;
 * dscale_pres: host, n_Q doubles of D_Q (> 0), or NULL. The library stores
 * D^{-1/2} on the device. All handles must live on the same device. */
fdp_status block_precond_setup(int D, const fdp_fd* vel, fdp_mass pres, const double* dscale_vel,
                               const double* dscale_pres, fdp_block* out);
int64_t block_precond_size(fdp_block h); /* sum_k N_k + n_Q */
size_t block_precond_workspace_bytes(fdp_block h, int64_t batch);
/* s = P_D^{-1} r (or (P_D^G)^{-1} r). r, s: device, batch*size doubles; s may alias r.
 * workspace: device, >= block_precond_workspace_bytes(h, batch) bytes (required, no internal
 * default). The launch sequence is captured once per (r, s, workspace, batch) into a CUDA graph
 * and replayed; if `stream` is being captured by the caller, kernels are launched directly. */
fdp_status block_precond_apply(fdp_block h, const double* r, double* s, int64_t batch,
                               void* workspace, void* stream);
/* End-to-end variant with HOST buffers (pinned recommended): copies r host->device, applies,
 * copies s device->host, and synchronises `stream` before returning. Uses handle-owned device
 * buffers sized on first use. */
fdp_status block_precond_apply_host(fdp_block h, const double* r_host, double* s_host,
                                    int64_t batch, void* stream);
/* Page-locked host memory for the host-buffer path (cudaMallocHost on the current device; H2D
 * from it runs at full PCIe rate). fdp_host_alloc returns NULL on failure (fdp_last_error says
 * why); fdp_host_free(NULL) is a no-op. */
void* fdp_host_alloc(size_t bytes);
fdp_status fdp_host_free(void* p);
fdp_status block_precond_destroy(fdp_block h);

/* Number of kernel launches one block_precond_apply issues for `batch` (for accounting): exact
 * (the kernel nodes of the CUDA graph captured for an apply of that batch size) once such an apply
 * has run on the handle, else a static estimate of the pass structure. Returns 0 for a NULL
 * handle or batch <= 0, -1 on an internal error. */
int fdp_block_launch_count(fdp_block h, int64_t batch);

/* Diagnostics: the number of kernel launches since library load that took the TMA-fed folded
 * transform kernel K1t, and the number that took the round-1 cp.async folded
 * kernel K1f instead (operands no tensor map can describe, or FDP_NO_TMA=1). Host-side counters
 * of enqueued launches (a CUDA-graph replay does not count again). */
int64_t fdp_debug_k1_launches(int tma);

/* Per-launch timing of block_precond_apply (roofline diagnostics). With enable != 0 every later
 * apply records a CUDA event on its stream before each kernel launch and after the last one (the
 * events become nodes of the cached graph, which is re-captured when the flag changes).
 * block_precond_profile_read fills, for the most recent apply, up to `max` entries: kind (0 = K1
 * mode contraction, 1 = K2 diagonal scaling, 2 = K3 banded mass solve), elapsed milliseconds
 * between the launch's start event and the next event, and the launch's ALGORITHMIC flops and
 * DRAM bytes (flops 2*N*n_d per contracted element set; bytes = one read + one write of the
 * tensor, plus scale vectors). Returns the number of launches (or -1 on error); call it after
 * the apply's stream has been synchronised. Any array may be NULL. */
fdp_status block_precond_profile(fdp_block h, int enable);
int block_precond_profile_read(fdp_block h, int max, int32_t* kind, float* ms, double* flops,
                               double* bytes);

/* ------------------------------------------------------------------------------------------
 * Matrix-free sums of Kronecker products (the Stokes system blocks of the
 * GPU-resident MINRES), y = beta*y + alpha * sum_t c_t (F_{t,D} (x) ... (x) F_{t,1}) x, with
 * rectangular factors F_{t,d} (nout_d x nin_d) applied as mode products (eq. kronvec).
 * ------------------------------------------------------------------------------------------ */
typedef struct fdp_kron_s* fdp_kron;
/* factors: host, nterms*D pointers, term-major (factor of term t, direction d at t*D + d), each
 * column-major nout[d] x nin[d]; coef: nterms scalars. D in {2,3}, extents in [1, 2048]. */
fdp_status kron_op_setup(int D, int nterms, const int32_t* nin, const int32_t* nout,
                         const double* const* factors, const double* coef, int device,
                         fdp_kron* out);
size_t kron_op_workspace_bytes(fdp_kron h, int64_t batch);
/* x: device, batch items of prod(nin) doubles at stride xbs; y: device, prod(nout) at stride ybs
 * (must not overlap x). beta = 0 overwrites y (NaNs in y ignored). Asynchronous on `stream`. */
fdp_status kron_op_apply(fdp_kron h, const double* x, int64_t xbs, double* y, int64_t ybs,
                         double alpha, double beta, int64_t batch, void* workspace, void* stream);
fdp_status kron_op_destroy(fdp_kron h);
/* Several operators in few launches (batch 1): for every distinct output pointer Y among y[i],
 * Y = beta * Y + sum_{i : y[i] == Y} alpha[i] * ops[i] x[i]. All terms of all operators run as one
 * grouped launch per mode (independent problems), each writing a private partial; one summation
 * pass per distinct output then combines them (no read-modify-write races). workspace >=
 * kron_ops_workspace_bytes(nops, ops). x[i] must not overlap any y. */
size_t kron_ops_workspace_bytes(int nops, const fdp_kron* ops);
fdp_status kron_ops_apply(int nops, const fdp_kron* ops, const double* const* x, double* const* y,
                          const double* alpha, double beta, void* workspace, void* stream);

/* ---- Block-triangular and constrained preconditioners (§4; NEXT-2) ----
 * P_T = [[P_V, B^T], [0, -P_Q]] and P_C = [[P_V, B^T], [B, B P_V^{-1} B^T - P_Q]]
 * (P:612-618), applied as s = P^{-1} r with r, s device [u_1 | .. | u_D | p] (batch 1, must not
 * alias). P_V, P_Q (and their P^G diagonal scalings) are the blocks of `P`
 * (block_precond_setup); B[k] (pressure x velocity-k, i.e. nin = velocity-k extents, nout =
 * pressure extents) and BT[k] (its transpose) are kron_op handles of the system's divergence
 * blocks B_k, sign included. P_T: back substitution s_p = -P_Q^{-1} r_p, s_u = P_V^{-1}(r_u - B^T s_p).
 * P_C: the paper's factorization applied right to left, two P_V^{-1} per apply.
 * The pressure block uses the banded per-mode solves. Asynchronous on `stream`, no allocation,
 * graph-capturable. workspace >= block_tri_workspace_bytes(...) (0 on invalid arguments). */
enum { FDP_PREC_TRIANGULAR = 1, FDP_PREC_CONSTRAINED = 2 };
size_t block_tri_workspace_bytes(fdp_block P, int variant, const fdp_kron* B, const fdp_kron* BT);
fdp_status block_tri_apply(fdp_block P, int variant, const fdp_kron* B, const fdp_kron* BT,
                           const double* r, double* s, void* workspace, void* stream);

/* ---- Peer-store slab exchange (SURVEY.md §8(e) "fused variant") ----
 * Same phases and slab partition as fd_apply_slab / kron_mass_apply_slab, but each exchange is
 * fused into the contraction before it: the kernel's epilogue stores every element directly into
 * the destination rank's buffer (peer memory mapped with fdp_peer_open, P2P over NVLink), so there
 * is no pack / unpack pass and no separate collective. `peers`: DEVICE array of nranks pointers.
 *  phase 0: in = this rank's z-slab (n1, n2, nz) [pre-scaled by dscale]; modes 1-2; element
 *           (i1, i2, i3) lands in peers[h] = the y-slab buffer (n1, ny_h, n3) of the rank h owning
 *           i2, at (i1, i2 - y0_h, z0 + i3).
 *  phase 1: in = this rank's y-slab buffer (filled by every rank's phase 0); the mode-3 triple
 *           (Lambda^{-1} included); element (i1, i2, i3) lands in peers[g] = the z-slab buffer
 *           (n1, n2, nz_g) of the rank g owning i3, at (i1, y0 + i2, i3 - z0_g).
 *  phase 2: in = this rank's z-slab buffer (filled by every rank's phase 1); modes 2-1 backward
 *           [post-scaled by dscale] -> out (n1, n2, nz).
 * Between phases every rank must pass fdp_peer_barrier. workspace: fd_slab_workspace_bytes /
 * kron_mass_slab_workspace_bytes. out unused in phases 0-1, peers unused in phase 2. */
fdp_status fd_apply_slab_peer(fdp_fd h, int phase, int nranks, int rank, const double* in,
                              double* out, double* const* peers, const double* dscale,
                              void* workspace, void* stream);
fdp_status kron_mass_apply_slab_peer(fdp_mass h, int phase, int nranks, int rank,
                                     const double* in, double* out, double* const* peers,
                                     const double* dscale, void* workspace, void* stream);
/* Cross-rank barrier on `stream` (one warp): increments *counter (device, this rank's epoch),
 * release-stores it (system scope, after a system fence that orders this rank's earlier peer
 * stores) into flags[o][rank] for every rank o, then acquire-spins until flags[rank][0..nranks-1]
 * all reach it. flags: DEVICE array of nranks pointers to each rank's nranks-slot uint64 flag
 * array (zero-initialised, mapped with fdp_peer_open). nranks <= 32. Graph-capturable. */
fdp_status fdp_peer_barrier(unsigned long long* const* flags, unsigned long long* counter,
                            int nranks, int rank, void* stream);
/* Device buffers shareable with peer processes over CUDA IPC: fdp_peer_alloc (cudaMalloc,
 * zeroed) returns the pointer and a 64-byte handle; another process maps it with fdp_peer_open
 * (lazy peer access) and unmaps with fdp_peer_close; the owner frees with fdp_peer_free. */
fdp_status fdp_peer_alloc(size_t bytes, int device, void** dev_ptr, void* ipc_handle);
fdp_status fdp_peer_open(const void* ipc_handle, int device, void** dev_ptr);
fdp_status fdp_peer_close(void* dev_ptr);
fdp_status fdp_peer_free(void* dev_ptr);

/* ---- Sharded applies (SURVEY.md §8(b) multi-GPU row, §8(e) config 5) ----
 * Slab decomposition of the last axis: rank g of nranks owns planes fdp_slab_range(n3, nranks, g)
 * of every block (its z-slab, vec order); mode 3 runs on y-slabs between two all-to-all
 * exchanges. Two kinds of communicator (fdp_comm), freed with fdp_comm_destroy:
 *
 * NCCL (the paper-independent baseline): rank 0 calls fdp_nccl_unique_id (128
 * bytes, host), the caller distributes them (e.g. the torch.distributed store), every rank calls
 * fdp_comm_init(nranks, rank, id, device). libfdp loads NCCL at run time (libnccl.so.2; in a
 * process that imported torch, torch's copy): FDP_ERR_NCCL when it cannot be loaded or a call
 * fails (fdp_last_error has NCCL's message). The exchanges are grouped ncclSend / ncclRecv of the
 * packed slab pieces (one NCCL group per exchange for all blocks). Such a comm serves any handle:
 *   fd_apply_sharded: x = D^{-1/2} U Lambda^{-1} U^T D^{-1/2} b on this rank's z-slab (b, x,
 *     dscale: device, n1 n2 nz doubles; dscale = the slab's slice of the length-N D, or NULL;
 *     x must not alias b); workspace >= fd_sharded_workspace_bytes(h, c) (0 for a peer comm).
 *   block_precond_apply_sharded (below).
 *
 * Peer-store (the exchanges fused into the contraction epilogues), for one block preconditioner P
 * (D = 3):
 *   1. fdp_comm_create: allocates this rank's exchange buffers (per block a y-slab and a z-slab,
 *      plus an nranks-slot barrier flag array) and writes its blob of CUDA IPC handles
 *      (fdp_comm_blob_bytes(P, nranks) bytes, host memory owned by the caller);
 *   2. the caller all-gathers the blobs (e.g. torch.distributed; rank-major, host);
 *   3. fdp_comm_connect maps every peer's buffers (P2P over NVLink / NVSwitch).
 *   Phases are separated by fdp_peer_barrier kernels; no NCCL call in the apply.
 *
 * block_precond_apply_sharded applies P_D^{-1} (or (P_D^G)^{-1}: the block's D scalings, sliced
 * to the rank's slab) to this rank's slabs: r, s device, block_precond_sharded_size doubles laid
 * out [u_1 z-slab | .. | u_D z-slab | p z-slab]. In every phase the steps of all blocks run side
 * by side (step i of the velocity blocks is one grouped launch). No host synchronisation;
 * graph-capturable (NCCL: as NCCL's own calls are). Every rank must make the same calls in the
 * same order. A communicator is not thread- or stream-safe; destroy every CUDA graph that
 * captured an apply on an NCCL communicator before fdp_comm_destroy (NCCL's teardown waits for
 * the graphs' resources). workspace: device, >=
 * block_precond_sharded_workspace_bytes(P, c) (per-block regions; NCCL comms also hold the
 * send / receive slabs there). */
typedef struct fdp_comm_s* fdp_comm;
#define FDP_NCCL_ID_BYTES 128
/* Host only: per-peer element counts of exchange 1 (z-slab pieces -> y-slab) or 2 (the reverse)
 * of a block with extents dims[0..2] for rank `rank` of nranks, in rank order (send_counts,
 * recv_counts: host arrays of nranks). Exchange 1 sends rank h the planes i2 in its y-range of my
 * z-slab (dims[0] ny_h nz doubles, packed in rank order) and receives its z-planes of my y-range
 * (dims[0] ny nz_h). FDP_ERR_INVALID_ARG on bad arguments. */
fdp_status fdp_slab_exchange_counts(const int32_t* dims, int nranks, int rank, int exchange,
                                    int64_t* send_counts, int64_t* recv_counts);
fdp_status fdp_nccl_unique_id(void* id);
fdp_status fdp_comm_init(int nranks, int rank, const void* nccl_unique_id, int device, fdp_comm* out);
size_t fd_sharded_workspace_bytes(fdp_fd h, fdp_comm c);
fdp_status fd_apply_sharded(fdp_fd h, fdp_comm c, const double* b, double* x, const double* dscale,
                            void* workspace, void* stream);
size_t fdp_comm_blob_bytes(fdp_block P, int nranks);
fdp_status fdp_comm_create(fdp_block P, int nranks, int rank, fdp_comm* out, void* blob);
fdp_status fdp_comm_connect(fdp_comm c, const void* all_blobs);
int64_t block_precond_sharded_size(fdp_block P, int nranks, int rank);
size_t block_precond_sharded_workspace_bytes(fdp_block P, fdp_comm c);
fdp_status block_precond_apply_sharded(fdp_block P, fdp_comm c, const double* r, double* s,
                                       void* workspace, void* stream);
fdp_status fdp_comm_destroy(fdp_comm c);

/* ---- Geometry-aware pencils (§6 P:1048-1059 and Appendix; NEXT-3) ----
 * Host setup helpers (no device work). The pencils themselves are iga_mixed with weights at the
 * quadrature points (K_d = int tau_d b' b', M_d = int mu_d b b), solved by fd_setup / fd_apply.
 *
 * iga_geometry_coeffs: c_out[d * nq^D + i] = c^k_dd at grid point i (i1 fastest; every direction
 * uses the nq points x) of C_k^TH = (J^{-1} J^{-T} + D_k D_k^T) |det J|, D_k = J^{-1} e_k
 * (eq. (Q_TH), nu = 1), for k = 0..D-1. kind FDP_GEOM_IDENTITY (D = 2, 3) or
 * FDP_GEOM_ANNULUS (D = 3: G = ((1+eta1) cos(pi eta2/4), (1+eta1) sin(pi eta2/4), eta3), the
 * eighth of the thick annulus of P:1264-1268). Errors: FDP_ERR_INVALID_ARG, FDP_ERR_UNSUPPORTED.
 *
 * iga_separable_fit: c_d (D host arrays over the nq[0] x .. x nq[D-1] grid, i1 fastest, > 0)
 * ~ tau_d(i_d) prod_{m != d} mu_m(i_m) (Appendix), by log-domain alternating least
 * squares (N3-2): init mu = 1, tau_d = slice geometric means; per sweep tau_1..tau_D then
 * mu_1..mu_D by closed-form slice means; gauge geomean(mu_m) = 1; stop when the objective's
 * relative change <= tol or after max_sweeps. tau, mu: host, concatenated per direction
 * (sum nq doubles each); *sweeps (may be NULL) = sweeps done. FDP_ERR_INVALID_ARG on c <= 0. */
enum { FDP_GEOM_IDENTITY = 0, FDP_GEOM_ANNULUS = 1 };
fdp_status iga_geometry_coeffs(int kind, int D, int k, int nq, const double* x, double* c_out);
fdp_status iga_separable_fit(int D, const int32_t* nq, const double* const* c, int max_sweeps,
                             double tol, double* tau, double* mu, int* sweeps);

/* Diagonals (host output, vec order i1 fastest), for the diagonal scalings D_V = diag(A) /
 * diag(P^_V), D_Q = diag(Q) / diag(P_Q) of §6:
 * fd_operator_diagonal: diag(R), R = sum_d coef_d (M_D (x) .. K_d .. (x) M_1) of the handle's pencils;
 * kron_op_diagonal: diag(sum_t c_t F_tD (x) .. (x) F_t1) of a square operator (nin == nout),
 * else FDP_ERR_SHAPE. */
fdp_status fd_operator_diagonal(fdp_fd h, double* out);
fdp_status kron_op_diagonal(fdp_kron h, double* out);

/* ---- Device-resident MINRES (NEXT-1): the Paige-Saunders scalar recurrence on the GPU,
 * so whole iterations can be captured in a CUDA graph with no host synchronisation ----
 * fdp_vec_lincomb_dev: out = k[0] x + k[1] y + k[2] z, coefficients read from DEVICE memory k
 * (3 doubles); a term with coefficient exactly 0 (or a NULL vector) is skipped, so stale
 * vectors of a finished solve are never read into the result.
 * fdp_minres_scalars(phase, state, hist, hist_cap, stream): one thread on `stream` updates the
 * device `state` (>= 32 doubles):
 *   [0] beta1 [1] beta [2] oldb [3] dbar [4] epsln [5] phibar [6] cs [7] sn [8] alfa (caller's
 *   v.y) [9] dot (caller's r.P r) [10] itn [11] done [12] itn at convergence [13] tol (caller)
 *   [14] error flag (P not positive definite) [16..18] k_v [19..21] k_y1 [22..24] k_y2
 *   [25..27] k_w [28..30] k_x (lincomb_dev coefficient triples).
 * phase 0 = init from dot = r.P r; 1 = iteration start (k_v = 1/beta, k_y1 = -beta/oldb);
 * 2 = after alfa (k_y2 = -alfa/beta); 3 = after dot (rotation, k_w, k_x = phi, stopping test
 * phibar/beta1 <= tol sets done and itn-at-convergence; hist[itn] = phibar/beta1 when hist != NULL
 * and itn < hist_cap). After `done`, every coefficient that would change x is 0. */
fdp_status fdp_vec_lincomb_dev(const double* coef, const double* x, const double* y,
                               const double* z, double* out, int64_t n, void* stream);
fdp_status fdp_minres_scalars(int phase, double* state, double* hist, int hist_cap, void* stream);

/* ---- Device-resident GMRES (NEXT-2): indices and counts read from device memory, so whole
 * Arnoldi steps can be captured in one CUDA graph ----
 * fdp_vec_copy_indexed: out = V_{*idx}; fdp_vec_store_indexed: V_{*idx} = (*coef) w, skipped
 * when *coef == 0; fdp_vec_multidot_dev / fdp_vec_gemv_dev: as fdp_vec_multidot / fdp_vec_gemv
 * over m = min(*m, m_max) vectors (grids sized for m_max; workspace as for m_max).
 * fdp_gmres_scalars(phase, istate, dstate, H, ldh, h1, h2, hist, m_max): one thread.
 *   istate (int[5]): [0] j (next column) [1] done [2] iterations at convergence [3] j + 1 (the
 *     multidot count) [4] index of the next basis vector;
 *   dstate (double[8 + 3 (m_max + 1)]): [0] beta = ||P^{-1} b|| [1] tol (caller) [2] coefficient
 *     of the next basis vector [3] ||w||^2 (caller) [4] ||P^{-1} b||^2 (caller), then cs, sn, g;
 *   H: column-major (ldh >= m_max + 1), column j = the Arnoldi coefficients h1 + h2 (classical
 *     Gram-Schmidt, two passes) and ||w||, rotated into R by the stored Givens rotations;
 *   phase 0 = init, 1 = one step (no-op after done); stopping rule |g_{j+1}| / beta <= tol. */
fdp_status fdp_vec_copy_indexed(const double* V, int64_t ldv, const int* idx, double* out,
                                int64_t n, void* stream);
fdp_status fdp_vec_store_indexed(double* V, int64_t ldv, const int* idx, const double* w,
                                 const double* coef, int64_t n, void* stream);
fdp_status fdp_vec_multidot_dev(const double* V, int64_t ldv, const int* m, int m_max,
                                const double* w, int64_t n, double* h, void* workspace,
                                void* stream);
fdp_status fdp_vec_gemv_dev(const double* V, int64_t ldv, const int* m, int m_max,
                            const double* h, double alpha, double* w, double beta, int64_t n,
                            void* stream);
fdp_status fdp_gmres_scalars(int phase, int* istate, double* dstate, double* H, int ldh,
                             const double* h1, const double* h2, double* hist, int m_max,
                             void* stream);

/* ---- Arnoldi helpers for GMRES (Saad & Schultz) ----
 * V: m device vectors of length n with stride ldv >= n (V_j = V + j*ldv).
 * fdp_vec_multidot: h[j] = V_j . w for j < m into device h; deterministic (fixed grid, fixed
 * reduction order); workspace >= fdp_vec_multidot_workspace_bytes(m).
 * fdp_vec_gemv: w = beta*w + alpha * sum_j h[j] V_j, h device (m <= 6144). */
size_t fdp_vec_multidot_workspace_bytes(int m);
fdp_status fdp_vec_multidot(const double* V, int64_t ldv, int m, const double* w, int64_t n,
                            double* h, void* workspace, void* stream);
fdp_status fdp_vec_gemv(const double* V, int64_t ldv, int m, const double* h, double alpha,
                        double* w, double beta, int64_t n, void* stream);

/* Mixed univariate matrix out[i, j] = int wt(x) b_test_i^(dtest)(x) b_trial_j^(dtrial)(x) dx on
 * [0,1] over n_el uniform elements with q Gauss points per element (q <= 0: deg_test+deg_trial+1
 * ... exact for unweighted products). wq: weights at the points iga_quadrature returns (n_el*q)
 * or NULL for wt = 1. flags as iga_univariate (FDP_IGA_INTERIOR per space). out: host,
 * column-major n_test x n_trial. */
fdp_status iga_quadrature(int n_el, int q, double* x, double* w);
/* Diagonal-of-mass factor: out[i + n*g] = w_g b_i(x_g)^2 at the n_el*q element Gauss points of
 * iga_quadrature (column-major n x (n_el q), host), so that for a weight f sampled at the points
 * int f b_i^2 = sum_g out[i, g] f(x_g); tensor products of these factors give diagonals of
 * weighted multivariate mass matrices (the D_Q = diag(Q) / diag(P_Q) scaling of P:1039 with
 * Q = int nu^{-1} rho_i rho_j). out NULL: only *n_out. flags: FDP_IGA_INTERIOR. */
fdp_status iga_mass_diag_factor(int deg, int alpha, int n_el, int flags, int q, double* out,
                                int32_t* n_out);
fdp_status iga_mixed(int deg_test, int alpha_test, int flags_test, int deg_trial, int alpha_trial,
                     int flags_trial, int n_el, int dtest, int dtrial, int q, const double* wq,
                     double* out, int32_t* n_test, int32_t* n_trial);

/* Vector kernels for the GPU Krylov driver (device pointers, asynchronous):
 * result[0] = x . y (FP64, deterministic two-level reduction); out = a x + b y + c z (z may be
 * NULL, out may alias any input). */
fdp_status fdp_vec_dot(const double* x, const double* y, int64_t n, double* result, void* stream);
fdp_status fdp_vec_lincomb(double a, const double* x, double b, const double* y, double c,
                           const double* z, double* out, int64_t n, void* stream);

/* ------------------------------------------------------------------------------------------
 * Slab decomposition for multi-GPU application: the slowest axis i3
 * is partitioned over `nranks` ranks (even split, the first n mod G ranks own one more plane).
 * Modes 1-2 are local to an i3-slab; mode 3 runs on i2-slabs after an all-to-all exchange (done
 * by the caller, e.g. NCCL over NVLink through torch.distributed) and is followed by the reverse
 * exchange. Batch 1. Rank r's pieces:
 *   z-slab (n1, n2, nz_r), planes [z0_r, z0_r + nz_r);  y-slab (n1, ny_r, n3), i2 in [y0_r, ...).
 *   A "piece buffer" of rank g holds, for every rank h in order, the block
 *   [i3 local][i2 - y0_h][i1] of size n1*ny_h*nz_g at offset n1*nz_g*y0_h.
 * Exchange 1 sends piece h of every rank's forward output to rank h; concatenating what rank h
 * receives, in source-rank order, IS its y-slab. Exchange 2 sends the contiguous planes
 * [z0_g, z0_g+nz_g) of every y-slab back to rank g, forming rank g's piece buffer.
 * ------------------------------------------------------------------------------------------ */
fdp_status fdp_slab_range(int64_t n, int nranks, int rank, int64_t* lo, int64_t* len);

/* FD phases (D = 3): phase 0 (fwd): in = b z-slab, out = piece buffer, dscale = D^{-1/2} on the
 * z-slab or NULL; computes x_1 U_1^T, x_2 U_2^T. Phase 1 (mid): in = out = y-slab (in place);
 * computes x_3 U_3^T, / Lambda, x_3 U_3 (Algorithm 1 steps 2-4 on the mode-3 fibers).
 * Phase 2 (bwd): in = piece buffer received in exchange 2, out = x z-slab; computes x_2 U_2,
 * x_1 U_1 and the post-scaling. workspace >= fd_slab_workspace_bytes(h, nranks, rank). */
size_t fd_slab_workspace_bytes(fdp_fd h, int nranks, int rank);
fdp_status fd_apply_slab(fdp_fd h, int phase, int nranks, int rank, const double* in, double* out,
                         const double* dscale, void* workspace, void* stream);

/* Kronecker mass inverse phases (banded solves): phase 0: modes 1-2 on the z-slab
 * (pre-scaling) then pack; phase 1: mode 3 on the y-slab in place; phase 2: unpack (post-scaling
 * with dscale on the z-slab). */
size_t kron_mass_slab_workspace_bytes(fdp_mass h, int nranks, int rank);
fdp_status kron_mass_apply_slab(fdp_mass h, int phase, int nranks, int rank, const double* in,
                                double* out, const double* dscale, void* workspace, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* FDP_H_ */

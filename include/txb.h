/*
 * txb.h — C ABI of the B200-native thread-transposed element integrator.
 *
 * This is the drop-in boundary for the reference's compiled lane.  Every entry
 * point takes plain pointers and sizes (no torch / numpy types); a Python host
 * binds it with ctypes (paper_1607_04245_b200/_lib.py), and INTEGRATION.md
 * shows the ctypes stub the reference's own backend.py would add.
 *
 * Reference interfaces replaced (paths relative to /root/reference/pkg/src):
 *   txb_query              <- txfem/backend.py:38-52   compiled_kernel(form, n_q, aux)
 *   txb_integrate_cells    <- txfem/_kernels_cy.pyx:37-123 integrate_cells(...)
 *                             reached via txfem/backend.py:55-87 run_compiled(...)
 *                             and txfem/executor.py:109-114 _run_span(...)
 *   txb_integrate_cells_host  same call with HOST buffers (the reference's own
 *                             calling convention: numpy arrays in host memory)
 *   txb_integrate_mesh     <- txfem/executor.py:194-212 (geometry + gather + cast
 *                             + integrate_cells, fused into one kernel)
 *   txb_tile_counts / txb_tile_build / txb_integrate_mesh_tiled
 *                          <- the same call as txb_integrate_mesh (executor.py:194-212)
 *                             over cached cell tiles with batch-local vertex tables
 *   txb_gather_coefficients   <- txfem/mesh.py:202-217 gather_coefficients
 *   txb_scatter_add           <- txfem/mesh.py:220-234 scatter_add_element_vectors
 *   txb_scatter_add_slots     <- the same, vertices visited in element-row order
 *   txb_compute_geometry      <- txfem/mesh.py:150-190 compute_geometry
 *   txb_jit_compile / txb_jit_integrate
 *                          <- txfem/physics.py:260-304 user_form + the string-
 *                             injection sources (physics.py:110-168) and
 *                             txfem/codegen.py:50-256 generate_kernel_source,
 *                             executed by the python lane
 *                             txfem/_kernels_py.py:20-110 (f0, n_aux, grad a)
 *   txb_halo_*             <- the global assembly across partitions (executor.py:266,
 *                             mesh.py:220-234 np.add.at order) for cell-range
 *                             partitions: peer-memory pack-and-put + assembly
 *   txb_last_error         error text for the Python exception message
 *
 * Codes follow the reference (backend.py:26-27):
 *   form_code: 0 poisson (f1 = grad u), 1 poisson_varcoef (f1 = a grad u),
 *              2 elasticity (f1 = sym grad u)
 *   aux_mode : 0 none, 1 P0 (one value per cell), 2 P1 (one value per vertex
 *              of the cell)
 *   dtype_bytes: 4 (float32) or 8 (float64); every array of one call has it.
 *
 * Array layouts (C-contiguous), identical to _kernels_cy.pyx:40-48:
 *   basis (n_q, n_b), basis_der (n_q, n_b, dim), weights (n_q)   HOST pointers
 *     (tiny tabulation; copied into the kernel's parameter space per launch)
 *   inv_j (n, dim, dim) row-major, det_j (n), coeffs (n, n_b, n_comp),
 *   aux (n, 1) [mode 1] | (n, n_b, 1) [mode 2] | NULL [mode 0],
 *   out (n, n_b, n_comp): caller-allocated, fully overwritten, the only
 *     buffer written.
 *
 * Threading / ownership: stateless and reentrant; the device
 * call is asynchronous on `stream` (a cudaStream_t, NULL = legacy default),
 * allocates nothing and never synchronises.  Inputs are read-only.
 *
 * Numerics: every multiply and add rounds separately in the configured
 * precision, in the reference's pinned order (reference.py:10-19), so results
 * are bit-identical to the reference compiled lane for f32 and f64 and to
 * integrate_reference for f64.
 */
#ifndef TXB_H_
#define TXB_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Return codes (0 = success).  The Python host re-raises the matching
 * txfem.errors class (errors.py:4-42). */
#define TXB_OK              0
#define TXB_E_UNSUPPORTED  -1  /* configuration outside the kernel surface  -> ValueError */
#define TXB_E_SHAPE        -2  /* inconsistent sizes                          -> ShapeError */
#define TXB_E_CONFIG       -3  /* n_bl / n_cb / thread-limit violation        -> ConfigurationError */
#define TXB_E_CAPACITY     -4  /* shared-memory image exceeds the device      -> CapacityError */
#define TXB_E_ARG          -5  /* NULL pointer where data is required         -> ValueError */
#define TXB_E_CUDA         -6  /* CUDA runtime error (text in txb_last_error) -> RuntimeError */
#define TXB_E_ORIENTATION  -7  /* detJ <= 0 in txb_compute_geometry           -> OrientationError */
#define TXB_E_COMPILE      -8  /* user physics source does not compile (NVRTC) -> CodegenError */

#define TXB_MAX_DIM    3
#define TXB_MAX_BASIS  4
#define TXB_MAX_COMP   3
#define TXB_MAX_QUAD   8
#define TXB_THREAD_LIMIT 1024

/* ABI version (bumped on any signature change). */
int txb_abi_version(void);

/* Thread-local text of the last failure on this thread ("" if none). */
const char* txb_last_error(void);

/* Capability probe: TXB_OK if txb_integrate_cells covers the configuration,
 * TXB_E_UNSUPPORTED otherwise.  Same coverage as backend.compiled_kernel:
 * dim<=3, n_b=dim+1<=4, n_q<=8, n_comp 1 (forms 0,1) or dim (form 2), aux
 * required by form 1 and forbidden for forms 0, 2. */
int txb_query(int form_code, int aux_mode, int dtype_bytes, int dim, int n_q, int n_comp);

/* Launch geometry the integrator would use (for tests, bench and tuning).
 * n_bl / n_cb <= 0 select the tuned defaults.  Outputs may be NULL.
 *   n_bc        cells per batch  (= n_bl * n_b * n_q, paper §3)
 *   n_t         threads per CTA  (= n_bc * n_comp)
 *   stages      shared-memory ring depth of the batch loader
 *   smem_bytes  dynamic shared memory per CTA
 *   grid        CTAs launched for n_cells on the current device            */
int txb_launch_config(int form_code, int aux_mode, int dtype_bytes, int dim, int n_q,
                      int n_comp, int64_t n_cells, int n_bl, int n_cb,
                      int* n_bc, int* n_t, int* stages, int* smem_bytes, int* grid,
                      int* n_bl_used, int* n_cb_used);

/* Element integration over n_cells cells, DEVICE pointers for the per-cell
 * arrays, HOST pointers for basis / basis_der / weights. */
int txb_integrate_cells(int form_code, int aux_mode, int dtype_bytes, int dim, int n_b,
                        int n_q, int n_comp, int64_t n_cells,
                        const void* basis, const void* basis_der, const void* weights,
                        const void* inv_j, const void* det_j, const void* coeffs,
                        const void* aux, void* out, int n_bl, int n_cb, void* stream);

/* Same call with every array in HOST memory (pinned or pageable).  Copies
 * the inputs to the device, integrates and copies `out` back, pipelined in
 * cell pieces over two streams; returns after `out` is complete. */
int txb_integrate_cells_host(int form_code, int aux_mode, int dtype_bytes, int dim, int n_b,
                             int n_q, int n_comp, int64_t n_cells,
                             const void* basis, const void* basis_der, const void* weights,
                             const void* inv_j, const void* det_j, const void* coeffs,
                             const void* aux, void* out, int n_bl, int n_cb);

/* Element integration fused with the reference's host-side preparation
 * (txfem/executor.py:194-212: compute_geometry, gather_coefficients, cast):
 * per-cell element vectors straight from the mesh.  DEVICE pointers:
 *   vertices (n_vertices, dim) float64, cells int64 (n_cells, dim+1),
 *   coeffs_global (n_vertices * n_comp) in the run dtype, aux per cell as in
 *   txb_integrate_cells, out (n_cells, dim+1, n_comp).
 * inv_j / det_j: NULL to compute the geometry from the vertices (float64,
 * mesh.py:150-190 expression order, then cast), or the caller's geometry in
 * the run dtype.  bad_cell: NULL or a device int64 preset to -1 (all bits
 * set); lowered to the first cell with detJ <= 0 (OrientationError).
 * Needs the standard P1 tabulation with n_q <= 2 (TXB_E_UNSUPPORTED
 * otherwise: use the unfused entry points).  Bit-identical to
 * compute_geometry -> gather -> cast -> txb_integrate_cells.  n_bl <= 0:
 * tuned default.  Asynchronous on `stream`. */
int txb_integrate_mesh(int form_code, int aux_mode, int dtype_bytes, int dim, int n_q, int n_comp,
                       int64_t n_cells, int64_t n_vertices,
                       const void* basis, const void* basis_der, const void* weights,
                       const double* vertices, const int64_t* cells, const void* coeffs_global,
                       const void* inv_j, const void* det_j, const void* aux, void* out,
                       int64_t* bad_cell, int n_bl, void* stream);

/* ---- Tiled mesh integration -------------------------------------------
 * A mesh's cells cut into tiles of tile_cells consecutive cells, each with
 * the list of its distinct vertices (a per-mesh structure, built once on the
 * device and cached):
 *   records (n_tiles, vrec) int32: [count, 0, 0, 0, ids ascending..., 0...]
 *   local   (n_tiles * tile_cells, 4) uint8 (local_bytes 1: every count
 *           <= 256) or uint16 (2): each cell's vertex positions in its tile's
 *           list (2D: the 4th entry 0); both zero-initialised by the caller.
 * txb_tile_counts writes each tile's count (n_tiles int32; -1 for a tile
 * holding a vertex id outside [0, 2^31)) so the caller can size
 * vrec = 4 + max(count) rounded up to a multiple of 4; txb_tile_build
 * fills records and local.  Connectivity int64 (n_cells, dim+1), vertex ids
 * < 2^31, tile_cells * (dim+1) <= 1024.  Asynchronous on `stream`. */
int txb_tile_counts(int dim, int64_t n_cells, const int64_t* cells, int tile_cells, int32_t* counts,
                    void* stream);
int txb_tile_build(int dim, int64_t n_cells, const int64_t* cells, int tile_cells, int vrec, int local_bytes,
                   int32_t* records, void* local, void* stream);

/* txb_integrate_mesh over the tiles above (records / local 16-byte aligned):
 * per tile, each distinct vertex's coefficients (and, with inv_j = det_j =
 * NULL, coordinates: geometry computed in-kernel) are gathered ONCE into
 * shared memory and the cells read them through their local indices; given
 * geometry (inv_j / det_j in the run precision) streams with the batch.  tile_cells must be a
 * multiple of (dim+1)*n_q and of 32/n_q with at most 6 warp slices (3D: 128,
 * 2D: 96 or 192 for the midpoint rule).  Same results, bit for bit, as
 * txb_integrate_mesh with the same inv_j / det_j; bad_cell as there. */
int txb_integrate_mesh_tiled(int form_code, int aux_mode, int dtype_bytes, int dim, int n_q, int n_comp,
                             int64_t n_cells, int64_t n_vertices,
                             const void* basis, const void* basis_der, const void* weights,
                             const double* vertices, int tile_cells, const int32_t* records, int vrec,
                             const void* local, int local_bytes, const void* coeffs_global, const void* inv_j,
                             const void* det_j, const void* aux, void* out, int64_t* bad_cell, void* stream);

/* Test hook: the fused kernels' branch-free float64 geometry per cell
 * (reciprocal + one residual correction; ok[c] = 0 where a cell's scale is
 * outside the range where that is the correctly rounded quotient and the
 * kernels recompute it with division).  exact_zero = 1: zero numerators keep
 * their sign (the run-time compiled kernels' variant).  Device pointers,
 * asynchronous. */
int txb_debug_geometry_fast(int dim, int64_t n_cells, const double* vertices, const int64_t* cells,
                            double* inv_j, double* det_j, int32_t* ok, int exact_zero, void* stream);

/* Test hook: the float32 runs' branch-free geometry (float32 of the float64
 * quotient from one product by RN(1/det); ok[c] = 0 where a quotient is near a
 * float32 rounding midpoint or out of range and the kernels recompute it).
 * inv_j / det_j float32.  Device pointers, asynchronous. */
int txb_debug_geometry_fast32(int dim, int64_t n_cells, const double* vertices, const int64_t* cells,
                              float* inv_j, float* det_j, int32_t* ok, void* stream);

/* Gather per-cell coefficient blocks (device pointers):
 *   out[c][b][k] = global[cells[c][b] * n_comp + k],  cells int64 (n, n_b). */
int txb_gather_coefficients(int dtype_bytes, int64_t n_cells, int n_b, int n_comp,
                            const int64_t* cells, const void* global, void* out, void* stream);

/* Deterministic scatter-add (device pointers).  `offsets` (n_vertices+1) and
 * `incidence` (n_cells*n_b) are the vertex->(cell*n_b+b) CSR built by
 * txb_build_incidence, entries in ascending cell order, so every vertex sum
 * runs in the reference's np.add.at order (bit-identical). */
int txb_scatter_add(int dtype_bytes, int64_t n_vertices, int n_comp,
                    const int64_t* offsets, const int32_t* incidence,
                    const void* elem, void* out, void* stream);

/* The same sums with the vertices visited in SLOT order (their first incident
 * element row ascending, txb_build_scatter_order): slot t sums the list
 * slot_incidence[slot_offsets[t] .. slot_offsets[t+1]) -- the list of vertex
 * slot_vertex[t], unchanged -- into out[slot_vertex[t]].  Bit-identical to
 * txb_scatter_add; neighbouring threads read neighbouring element rows even
 * when the mesh numbers vertices and cells in different orders. */
int txb_scatter_add_slots(int dtype_bytes, int64_t n_vertices, int n_comp,
                          const int64_t* slot_offsets, const int32_t* slot_incidence,
                          const int32_t* slot_vertex, const void* elem, void* out, void* stream);

/* Slot order of a vertex CSR (offsets/incidence from txb_build_incidence,
 * n_entries = offsets[n_vertices]): slot_vertex (n_vertices), slot_offsets
 * (n_vertices+1), slot_incidence (n_entries).  `scratch` needs
 * txb_scatter_order_scratch_bytes(n_vertices) bytes. */
int64_t txb_scatter_order_scratch_bytes(int64_t n_vertices);
int txb_build_scatter_order(int64_t n_vertices, int64_t n_entries, const int64_t* offsets,
                            const int32_t* incidence, int64_t* slot_offsets, int32_t* slot_incidence,
                            int32_t* slot_vertex, void* scratch, void* stream);

/* Build the vertex incidence CSR on the device from the connectivity
 * (cells int64 (n, n_b)).  `offsets` has n_vertices+1 entries, `incidence`
 * n_cells*n_b; `scratch` needs txb_incidence_scratch_bytes(...) bytes. */
int64_t txb_incidence_scratch_bytes(int64_t n_cells, int n_b, int64_t n_vertices);
int txb_build_incidence(int64_t n_cells, int n_b, int64_t n_vertices, const int64_t* cells,
                        int64_t* offsets, int32_t* incidence, void* scratch, void* stream);

/* Per-cell inverse Jacobians and determinants from vertex coordinates
 * (device pointers, float64 like mesh.compute_geometry).  Returns
 * TXB_E_ORIENTATION (and sets *bad_cell, a host pointer) when some
 * detJ <= 0; synchronises on `stream` to read the flag. */
int txb_compute_geometry(int dim, int64_t n_cells, const double* vertices, const int64_t* cells,
                         double* inv_j, double* det_j, int64_t* bad_cell, void* stream);

/* ---- Run-time compiled user physics (NVRTC, sm_100a) -------------------
 * The form's pointwise functions are source text in the reference's
 * string-injection dialect (physics.py:110-112): real / realv (d-vector with
 * .x .y [.z]) and
 *   realv f1_<name>(const real u[], const realv gradU[], const real a[],
 *                   const realv gradA[], int comp)
 *   real  f0_<name>(...same arguments...)          (optional: source_f0 NULL)
 * txb_jit_compile assembles the integration kernel around them (the batch
 * pipeline of txb_integrate_cells; every chain in the numpy lane's order,
 * _kernels_py.py:20-110, compiled with -fmad=false), compiles it with NVRTC
 * and returns a process-lifetime handle (memoised on the generated text; no
 * device needed).  aux_mode 0/1/2 = none/P0/P1 with n_aux fields (1..4; 0
 * iff aux_mode 0); P0 aux (n, n_aux), P1 aux (n, n_b, n_aux); uses_grad_a
 * computes gradA for P1 (zero otherwise, _kernels_py.py:93-110).
 * TXB_E_COMPILE carries the NVRTC log in txb_last_error. */
int txb_jit_compile(const char* name, const char* source_f1, const char* source_f0, int dtype_bytes,
                    int dim, int n_q, int n_comp, int n_aux, int aux_mode, int uses_grad_a,
                    void** kernel);

/* The generated translation unit and the compiler log of a handle. */
const char* txb_jit_source(void* kernel);
const char* txb_jit_log(void* kernel);
int64_t txb_jit_cubin_bytes(void* kernel);
/* Copies the sm_100a cubin into dst when capacity suffices; returns its size. */
int64_t txb_jit_cubin(void* kernel, void* dst, int64_t capacity);

/* txb_integrate_cells for a run-time compiled form: same layouts, device
 * pointers, host tables, asynchronous on `stream`; the first call on a
 * device loads the module there. */
int txb_jit_integrate(void* kernel, int64_t n_cells, const void* basis, const void* basis_der,
                      const void* weights, const void* inv_j, const void* det_j, const void* coeffs,
                      const void* aux, void* out, int n_bl, int n_cb, void* stream);

/* The run-time compiled form on a mesh, fused like txb_integrate_mesh: device
 * vertices (n_vertices, dim) float64, cells int64 (n_cells, dim+1),
 * coeffs_global (n_vertices * n_comp) in the kernel's precision, per-cell aux
 * as in txb_jit_integrate; the float64 geometry (cast once) and the gather
 * run in-kernel; bad_cell as for txb_integrate_mesh.  Any tabulation. */
int txb_jit_integrate_mesh(void* kernel, int64_t n_cells, int64_t n_vertices, const void* basis,
                           const void* basis_der, const void* weights, const double* vertices,
                           const int64_t* cells, const void* coeffs_global, const void* aux, void* out,
                           int64_t* bad_cell, int n_bl, void* stream);

/* The run-time compiled form over cell tiles (txb_tile_build tables), like
 * txb_integrate_mesh_tiled: each tile's distinct vertex rows gathered once
 * into shared memory; inv_j / det_j NULL (geometry in-kernel, same bits as
 * txb_jit_integrate_mesh) or the caller's geometry in the kernel's precision
 * (same bits as gather + txb_jit_integrate).  n_q <= 2; tile_cells a
 * multiple of (dim+1)*n_q and of 32/n_q with at most 8 warp slices. */
int txb_jit_integrate_mesh_tiled(void* kernel, int64_t n_cells, int64_t n_vertices, const void* basis,
                                 const void* basis_der, const void* weights, const double* vertices,
                                 int tile_cells, const int32_t* records, int vrec, const void* local,
                                 int local_bytes, const void* coeffs_global, const void* inv_j, const void* det_j,
                                 const void* aux, void* out, int64_t* bad_cell, void* stream);

/* ---- Halo exchange over peer memory (one node, NVLink / NVSwitch) --------
 * The global-residual exchange of halo.py without NCCL: every rank exposes a
 * WINDOW (header of epoch flags/acks + two receive slots of n_recv rows), shared
 * with the other processes by CUDA IPC handle (64 bytes).  Per residual
 * evaluation (epoch 1, 2, ...):
 *   txb_halo_put       stores this rank's owed rows straight into each owner's
 *                      window (P2P), then publishes the epoch in the owners'
 *                      flags (release, system scope); waits for the owner's ack
 *                      of epoch-2 before reusing a slot;
 *   txb_halo_assemble  waits until every sender's flag reached the epoch, runs
 *                      the CSR chain over [local rows | received rows]
 *                      (txb_scatter_add's np.add.at order), acks the epoch.
 * `windows` is a DEVICE array of `world` window pointers valid in this process
 * (own window + opened peers); `slot_bytes` a device array of each window's
 * slot size.  Spins time out after TXB_HALO_TIMEOUT_MS (default 10 s) and
 * record an error instead of hanging (txb_halo_window_error). */
int64_t txb_halo_window_bytes(int64_t n_recv_rows, int n_comp, int dtype_bytes);
int txb_halo_window_alloc(int64_t bytes, void** window, void* ipc_handle);
int txb_halo_window_open(const void* ipc_handle, void** window);
int txb_halo_window_close(void* window);
int txb_halo_window_free(void* window);
int txb_halo_window_error(void* window, int* error);
int txb_halo_put(int dtype_bytes, int n_comp, int rank, int world, int64_t n_send,
                 const int64_t* send_rows, const int32_t* send_peer, const int64_t* send_dst,
                 const void* elem, void* const* windows, const int64_t* slot_bytes,
                 const int32_t* out_peers, int n_out_peers, uint64_t epoch, void* stream);
int txb_halo_assemble(int dtype_bytes, int n_comp, int rank, int world, int64_t n_owned,
                      const int64_t* offsets, const int32_t* incidence, int64_t n_local_rows,
                      const void* elem, void* const* windows, int64_t my_slot_bytes,
                      const int32_t* in_peers, int n_in_peers, uint64_t epoch, void* out, void* stream);

/* Debug timeline of txb_integrate_cells launches made by THIS thread: each
 * later launch takes the next 4*grid u64 of `device_buf` (capacity in u64) and
 * its CTAs write %globaltimer stamps [entry, after the previous-grid wait,
 * first batch ready (only in builds with -DTXB_TRACE_FIRST_BATCH, else 0),
 * consumers done].  NULL turns it off.  Tuning aid only. */
int txb_debug_trace(void* device_buf, int64_t capacity_u64);

/* STREAM-like probe at a given read:write byte ratio (device pointers):
 * reads `read_bytes` from src, writes `write_bytes` to dst, 16-byte vector
 * accesses.  Used by bench.py for the "measured achievable" bandwidth. */
int txb_stream_probe(const void* src, int64_t read_bytes, void* dst, int64_t write_bytes,
                     void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TXB_H_ */

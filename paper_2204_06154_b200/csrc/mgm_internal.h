// Internal declarations of libmgm (not part of the ABI).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

namespace mgm {

using i64 = int64_t;
using i32 = int32_t;

// Device memory of a ctx (setup scratch included) goes through the allocator passed to
// mgm_setup (include/mgm.h mgm_allocator; NULL = cudaMalloc / cudaFree).  The current
// allocator is thread-local: every ABI entry point installs its ctx's (AllocScope).
cudaError_t dev_malloc(void** p, size_t bytes);
void dev_free(void* p);

// Host CSR (int64 row pointer, int32 columns ascending within a row).
struct HostCSR {
    i64 nrows = 0, ncols = 0;
    std::vector<i64> ptr;
    std::vector<i32> col;
    std::vector<double> val;
    i64 nnz() const { return ptr.empty() ? 0 : ptr.back(); }
};

// ---------------- host setup (host_setup.cpp; compiled with -ffp-contract=off) ----------
// Morton permutation (O1): perm[new] = old.  Returns false on a degenerate cloud.
bool morton_order(const double* pts, i64 n, std::vector<i64>& perm);

// k nearest neighbours of each query among `pts` under the (d2, index) order of O2.
// out[q*k + t] (int32 indices into pts).  Multi-threaded, exact.
void knn_grid(const double* pts, i64 n, const double* qry, i64 nq, int k, std::vector<i32>& out,
              int nthreads);

// Duplicate check: returns the index of a point whose nearest other point is at distance 0,
// or -1.  nn2[i] receives the squared distance to the nearest other point.
i64 nearest_other(const double* pts, i64 n, std::vector<double>& nn2, int nthreads);

// Weighted sample elimination (O8): keep (size nt) = surviving indices, ascending.
double wse_initial_radius(const std::vector<double>& nn2, i64 n, i64 nt);
void wse_eliminate(const double* pts, i64 n, i64 nt, const std::vector<double>& nn2,
                   std::vector<i64>& keep, int nthreads);

// Greedy colouring (O11) of sym(pattern(A)) minus the diagonal in index order.
// device >= 0: the iterated-greedy passes run on that GPU (ig_passes_device) for patterns of
// at least MGM_IG_DEVICE_MIN (default 65536) rows -- the same colours.
int greedy_colouring(const HostCSR& A, std::vector<i32>& colour, int passes, int device = -1);
// Iterated-greedy passes on the device from a colouring with ncol <= 255 colours (host CSR
// adjacency in, colours in/out): the new colour count, or -cudaError_t.
int ig_passes_device(i64 n, const i64* np, const i32* nb, i32* colour, int ncol, int passes, int device);
// O11 iterated-greedy passes: 10, or MGM_COLOUR_PASSES (experiments; the oracle must match)
int colour_passes();

HostCSR transpose(const HostCSR& A);

// Dense LU with partial pivoting (ties -> lowest row), column-major output for the device
// solve.  Returns -1 on success or the failing pivot column.
i64 dense_lu_colmajor(std::vector<double>& A_rowmajor, int m, std::vector<double>& LU_colmajor,
                      std::vector<i32>& piv);
// Explicit inverse (row-major) from those factors, columns on `nthreads` threads.
void dense_inverse(const std::vector<double>& LU, const std::vector<i32>& piv, int m, std::vector<double>& Ainv,
                   int nthreads);

// ---------------- distributed solve: partition of one level (host_setup.cpp) ------------
// SURVEY 8(e) / DESIGN.md "Multi-GPU": rank q owns the rows with owner[r] == q (a Morton
// block); its vectors hold [owned rows | (Poisson multiplier) | ghost rows].  A ghost is a
// row another rank owns whose value one of q's operator applications reads:
//   * columns of L_j in q's rows (Gauss-Seidel, residual, SpMV),
//   * fine columns (level j) of R_j = P_j^T in the coarse rows q owns at level j+1,
//   * coarse columns (level j) of P_{j-1} in the fine rows q owns at level j-1.
// Ghosts are sorted by (owner, row); rows are in lib order (colour-major), so the ghosts a peer
// sends for one colour are a contiguous slice of the segment from that peer -- a per-colour
// halo is one send / one receive per peer, received straight into the ghost slots.
struct PartTables {
    std::vector<i64> rows;              // owned rows (ascending)
    std::vector<i64> ghosts;            // ghost rows, sorted by (owner, row)
    std::vector<int> peers;             // ranks q exchanges with (ascending)
    std::vector<i64> send_rows;         // per peer (concatenated): owned rows that peer needs, ascending
    std::vector<i64> send_off, recv_off;  // per peer: offsets into send_rows / ghost slots (npeers + 1)
    std::vector<i64> send_coff, recv_coff;  // [npeers][ncol + 1]: absolute offsets of each colour's slice
};
// need[p] = rows of this level that rank p reads (owned or not), from the three operators
// above; the helper collects them for every rank at once (O(nnz)).
// L: this level's operator (lib order, n rows); owner[n]; colour[n] (ncol colours);
// Rt: P_j (fine rows n -> coarse cols), owner_c[nc] of level j+1 rows (or NULL on the coarsest
// distributed level's absent transfer); Pf: P_{j-1} (fine rows nf of level j-1 -> cols of this
// level), owner_f[nf] (or NULL on level 0).
void partition_level(const HostCSR& L, const std::vector<int>& owner, const std::vector<i32>& colour, int ncol,
                     const HostCSR* Pj, const std::vector<int>* owner_c, const HostCSR* Pf,
                     const std::vector<int>* owner_f, int nranks, std::vector<PartTables>& out);

// ---------------- device setup kernels (setup_kernels.cu; -fmad=false) -----------------
// All pointers device.  Return cudaError_t as int; *fail_dev = failing row or INT64_MAX.
int launch_rbffd_weights(const double* pts, const double* nrm, const i32* sten, i64 n, int ns,
                         int ell, int k, double* w, i64* fail_dev, void* stream);
int launch_stencil_radius(const double* pts, const double* nrm, const i32* sten, i64 n, int ns,
                          double* rho, void* stream);
int launch_gfd_weights(const double* pts, const double* nrm, const i32* sten, i64 n, int ns,
                       int ell, double alpha, const double* rho, double* w, i64* fail_dev,
                       void* stream);
int launch_interp_weights(const double* fine, i64 nf, const double* coarse, const i32* sten,
                          int m, double* w, i32* cnt, i64* fail_dev, void* stream);

// Exact kNN on the device (same lists as knn_grid; k <= 64).  h_pts: the same points on the
// host (bounding box); d_out[nq * k].  Synchronises the stream.
int knn_device(const double* h_pts, const double* d_pts, i64 n, const double* d_qry, i64 nq, int k, i32* d_out,
               void* stream);

// nearest_other on the device (the same nn2 bits; k = 3 lists from knn_device): the smallest
// duplicate index or -1; *err a cudaError_t.
i64 nearest_other_device(const double* h_pts, const double* d_pts, i64 n, std::vector<double>& nn2, void* stream,
                         int* err);

// Weighted sample elimination (O8) on the device: the same survivors as wse_eliminate (same
// neighbour sets and fixed-point weights, the same rounds of local maxima, the same final
// selection).  d_pts: the n points on the device; nn2: nearest-other squared distances (host).
// keep: ascending survivor indices.  Synchronises the stream; returns a cudaError_t.
int wse_device(const double* d_pts, const double* h_pts, i64 n, i64 nt, const std::vector<double>& nn2,
               std::vector<i64>& keep, void* stream);

// Device SpGEMM C = A B (CSR, columns ascending).  Symbolic pattern kept in full; values
// summed in canonical order (O10), bit-identical to a sequential loop.
struct DevCSR {
    i64 nrows = 0, ncols = 0, nnz = 0;
    i64* ptr = nullptr;
    i32* col = nullptr;
    double* val = nullptr;
};
int spgemm_device(const DevCSR& A, const DevCSR& B, DevCSR& C, void* stream, std::string& err);
void free_dev_csr(DevCSR& M);
int upload_csr(const HostCSR& H, DevCSR& D, void* stream);
int download_csr(const DevCSR& D, HostCSR& H, void* stream);

}  // namespace mgm

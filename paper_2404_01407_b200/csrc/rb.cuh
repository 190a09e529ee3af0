// rb.cuh -- the 2-colour ("red-black") fast path of ILU(0)-Richardson.
//
// With a colour-major ordering of a 2-colourable graph (every hex mesh) and a single
// partition, the reference ILU(0) (sparse.cpp:187-291) has a closed form:
//   colour 0 rows (first N0):  no lower entries; U_ij = A_ij; pivot = A_ii + s_i
//   colour 1 rows:             L_ik = A_ik * inv(U_kk) (k colour 0); U_ii = A_ii + s_i
//                              - sum_k L_ik A_ki; no upper entries
// so the factorization stores only the pivot LUs (and inv(U_kk) for colour 0) and
// the sweep recomputes L_ik = A_ik * inv(U_kk) from the shared real LHS A5 with the
// reference's own operation order: the iterates are bitwise those of
// smoothed_solve (sparse.hpp:295-331), only the residual-norm summation order
// differs.  One sweep = three kernels:
//   K_F(s)  colour 1: forward substitution with L = A inv(U) + pivot solve
//   K_B(s)  colour 0: backward substitution + x += z + residual rows, one pass over A
//   K_R(s)  colour 1: x += z + residual rows + norm / stopping decision (last CTA)
// (colour-1 blocks are read twice, colour-0 blocks once).  A5 is stored SELL-32
// (slice of 32 rows, slot-major, lane-minor) so each warp load is 256 contiguous
// bytes.  The stopping rule is evaluated on the device: no host round trip per sweep.
#pragma once

#include "capi_util.hpp"
#include "la.cuh"

namespace fnlh {

// SELL-32 copy of a BSR on a colour-major 2-colour pattern
struct SellLayout {
    int n = 0, n0 = 0, b = 0;
    int nslices = 0;
    DeviceBuffer<long long> slice_val;   // element offset of slice s in vals
    DeviceBuffer<int> slice_col;         // entry offset of slice s in cols
    DeviceBuffer<int> deg;               // per row: number of entries
    DeviceBuffer<int> dslot;             // per row: slot of the diagonal
    DeviceBuffer<int> cols;              // [slice][slot][lane]
    DeviceBuffer<long long> csr_to_sell; // per CSR entry: element offset of its block's k = 0 entry
    long long total_vals = 0;               // doubles per scalar component (incl. padding)
    int slice_of_row0 = 0;                  // first slice of colour 1
};

struct RbControl {  // device-side Richardson control block
    double target;
    double initial_residual;
    double final_residual;
    int iterations;
    int converged;
    int done;
    int status;  // 0 ok, 6 divergence (non-finite)
    unsigned int counter;
    int pad;
};

// global switch (fnlh_set_red_black) so tests can force the general level-scheduled path
inline std::atomic<bool>& rb_enabled() {
    static std::atomic<bool> on{true};
    return on;
}
// fnlh_set_rb_sweep: the 2-colour sweep variant
//   0 (default) reference operation order, K_R(s) fused with K_F(s+1): 2 kernels per sweep
//   1           reference operation order, split K_F / K_B / K_R: 3 kernels per sweep
//   2           one pass over A per sweep, L_ik r_k applied as A_ik (U_kk^{-1} r_k):
//               same preconditioner, iterates equal to rounding (not bitwise)
inline std::atomic<int>& rb_sweep_mode() {
    static std::atomic<int> mode{0};
    return mode;
}

// is the pattern a 2-colour colour-major ordering with one partition?
bool rb_eligible(const DevicePattern& p, int* n0);

// element (m, c) of node k's inv(U_kk) block in RbIlu::inv0 (slice-major; rb.cu ubase / uix)
inline std::size_t rb_uoff(int b, int k, int m, int c) {
#ifdef RB_U_AOS
    return (std::size_t)k * b * b + m * b + c;
#else
    return (std::size_t)(k >> 5) * 32 * b * b + (std::size_t)(m * b + c) * 32 + (k & 31);
#endif
}

template <class S>
struct RbIlu {
    const DevicePattern* p = nullptr;
    int n0 = 0;
    S* diag_lu = nullptr;   // pivot LUs, slice-major [slice][k][lane] (rows padded to 32 per colour)
    int* diag_piv = nullptr;  // same layout, b per row
    S* inv0 = nullptr;      // inv(U_kk) of colour 0 rows, slice-major [slice][element][lane] (rb_uoff), rows padded to 32
    RbIlu(const DevicePattern* pat, int n0_);
    ~RbIlu();
    RbIlu(const RbIlu&) = delete;
    RbIlu& operator=(const RbIlu&) = delete;
    std::size_t bytes() const;
    std::size_t packed_rows() const {
        return (std::size_t)32 * ((n0 + 31) / 32 + (p->rows - n0 + 31) / 32);
    }
    // packed row index of row i, element stride 32 (host-side unpacking)
    std::size_t packed_base(int i, int width) const {
        const int li = i < n0 ? i : i - n0;
        const std::size_t s = (i < n0 ? 0 : (n0 + 31) / 32) + (li >> 5);
        return s * 32 * width + (li & 31);
    }
};

class RbSystem {
public:
    RbSystem(const DevicePattern* p, int n0);
    // A5 (CSR layout, p's pattern) -> SELL copy
    void load(const double* A_csr, cudaStream_t st);
    const SellLayout& layout() const { return L_; }
    const double* vals() const { return vals_.ptr; }
    double* vals_mut() { return vals_.ptr; }
    const long long* sell_map() const { return L_.csr_to_sell.ptr; }
    std::size_t bytes() const { return vals_.bytes(); }
    int n0() const { return L_.n0; }
    const DevicePattern* pattern() const { return p_; }

private:
    const DevicePattern* p_;
    SellLayout L_;
    DeviceBuffer<double> vals_;
    DeviceBuffer<long long> trans_;  // per CSR entry (i,k): SELL offset of the (k,i) block
public:
    DeviceBuffer<double> partials;   // per-CTA norm partials (colour 0 then colour 1)
    std::size_t partials_len() const { return partials.n; }
    int grid0 = 0, grid1 = 0;
    const long long* trans() const { return trans_.ptr; }
};

// factorize the (shifted) system into the compact RB factors; throws FactorizationError
template <class S>
void rb_factorize(const RbSystem& A, const double* shift_im, RbIlu<S>& f, Workspace& ws);
// same, enqueued only: status[1] receives the first near-singular pivot row (0x7fffffff when clean)
template <class S>
void rb_factorize_async(const RbSystem& A, const double* shift_im, RbIlu<S>& f, int* status, cudaStream_t st);

constexpr int kMaxBatch = 8;

// one system of a batched solve: its factors, shift, vectors and control block
template <class S>
struct RbMember {
    const RbIlu<S>* f;
    const double* shift;  // shift_im (complex systems) or nullptr
    const S* rhs;
    S* x;
    S* z;
    S* r;
    RbControl* ctl;
    double* partials;  // >= RbSystem::partials_len() doubles
};

// enqueue P independent smoothed_solves on systems sharing A (one CTA stream per member,
// interleaved so A is fetched from HBM once per batched sweep); each member stops on
// its own rule; reports land in mem[m].ctl
template <class S>
void rb_smoothed_solve_batch(const RbSystem& A, const RbMember<S>* mem, int P, double tol_rel, int max_iter,
                             cudaStream_t st);

// enqueue a complete smoothed_solve (no host synchronization); the report lands in *ctl
// (device); x is overwritten.
template <class S>
void rb_smoothed_solve(const RbSystem& A, const double* shift_im, const RbIlu<S>& f, const S* rhs, double tol_rel,
                       int max_iter, S* x, S* z, S* r, RbControl* ctl, Workspace& ws);

}  // namespace fnlh

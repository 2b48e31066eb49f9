// Multi-GPU CN-WSGD time step by y-slab decomposition, host
// side in C++.  One rank per GPU owns grid rows [r0, r1) of every slab level:
//
//   * row (x-direction) Toeplitz lines are slab-local;
//   * the column pass is an all-to-all transpose, the column kernels on the
//     columns the rank then owns, and an all-to-all back
//     (structured.cpp:139-147 distributed);
//   * restriction / prolongation along y read one halo row per neighbour;
//   * levels below `agglomerate` unknowns are replicated: the restricted
//     right-hand side is all-gathered and every rank runs the rest of the
//     V-cycle locally (multigrid.cpp:318-383), so the coarse tail pays no
//     collective latency;
//   * Krylov inner products are local partials, all-gathered and summed in
//     rank order on the device (the same bits on every rank); the host reads
//     one small block per Arnoldi step, as the single-GPU gmres does
//     (krylov.cpp:89-130).
//
// The transport is a SlabComm: NCCL (one process per GPU; libnccl is opened
// at run time, so the library itself has no link dependency on it) or
// in-process virtual ranks (P host threads sharing one device and one stream:
// the same solver code, collectives as ordered device copies -- how the
// N > 1 code paths are exercised on a single GPU).
#pragma once
#include <memory>
#include <vector>

#include "krylov.cuh"
#include "problem.cuh"
#include "slab.cuh"

namespace fde_b200 {

class SlabComm {
 public:
  virtual ~SlabComm() = default;
  int rank() const { return rank_; }
  int world() const { return world_; }
  // element counts per peer; chunks are contiguous in rank order on both sides
  virtual void all_to_all(const double* send, const size_t* scnt, double* recv,
                          const size_t* rcnt, cudaStream_t s) = 0;
  // recv[q * count .. ) = rank q's `count` doubles
  virtual void all_gather(const double* send, double* recv, size_t count, cudaStream_t s) = 0;
  // rank q contributes counts[q] doubles; recv is their concatenation in rank order
  virtual void all_gather_v(const double* send, double* recv, const size_t* counts,
                            cudaStream_t s) = 0;
  // one row of `width` doubles to / from each neighbour: send_down goes to
  // rank - 1 (its `above`), send_up to rank + 1 (its `below`); null = none
  virtual void halo(const double* send_down, const double* send_up, double* below, double* above,
                    size_t width, cudaStream_t s) = 0;
  // whether the collectives may be recorded into a CUDA graph
  virtual bool capturable() const = 0;
  unsigned long long collectives() const { return ncoll_; }

 protected:
  int rank_ = 0, world_ = 1;
  unsigned long long ncoll_ = 0;
};

// NCCL transport.  id128: the 128-byte ncclUniqueId made by nccl_unique_id()
// on one rank and handed to the others by the launcher.
void nccl_unique_id(void* id128);
std::shared_ptr<SlabComm> make_nccl_comm(const void* id128, int rank, int world);
// P virtual ranks of one process (every rank must run on its own host thread
// and enqueue on the same stream).
std::vector<std::shared_ptr<SlabComm>> make_virtual_comms(int P);
// wake the other virtual ranks with an error after one of them failed
void abort_virtual(SlabComm& c);

std::vector<size_t> split_ranges(size_t n, int parts);
// coarse row b belongs to the rank that owns its centre fine row 2b + 1 - par
std::vector<size_t> induced_coarse_rows(const std::vector<size_t>& fine_offsets, size_t d2,
                                        bool coarsen_y);

// Rank-local piece of one level operator and its transpose plumbing.
class DistLevel {
 public:
  DistLevel(SlabComm& c, const Problem& p, size_t nf1, size_t nf2, size_t d1, size_t d2,
            std::vector<size_t> row_offsets, size_t steps, size_t m);
  size_t local_size() const { return nr * d1; }
  // out = epilogue(A x) on the rank's rows (SlabOp::xpass epilogues)
  void run(const double* x, double* out, double sign, int epi, const EpiArgs& e,
           cudaStream_t s, const InMap* in = nullptr);
  SlabComm& comm;
  size_t d1, d2, r0, r1, c0, c1, nr, nc;
  std::vector<size_t> rows, cols;
  DevBuf<double> dinv;

 private:
  std::unique_ptr<SlabOp> op_;
  DevBuf<double> xTl_, recv_, xT_, QT_, send2_, recv2_, Q_;
  std::vector<size_t> s1_, r1_, s2_, r2_;
  std::vector<long long> rows_ll_;
};

// Geometric V(1,1) cycle over slab levels with the replicated coarse tail.
class DistHierarchy {
 public:
  DistHierarchy(SlabComm& c, const Problem& p, size_t n1, size_t n2, size_t steps, size_t m,
                double omega, int coarse, size_t coarse_sweeps, size_t agglomerate,
                std::shared_ptr<DistLevel> fine);
  // x = V-cycle(b) from a zero guess (Precond::apply with cycles = 1)
  void vcycle(const double* b, double* x, cudaStream_t s);
  size_t slab_levels() const { return levels_.size(); }
  const std::vector<std::pair<size_t, size_t>>& dims() const { return dims_; }

 private:
  void cycle(size_t l, const double* b, double* x, bool zero, cudaStream_t s);
  void sweep(size_t l, const double* b, double* x, cudaStream_t s);
  void restrict_to(size_t l, const double* r_local, double* out, size_t c_lo, size_t c_hi,
                   cudaStream_t s);
  void prolong_add(size_t l, const double* xc_local, double* x, cudaStream_t s);
  void record(const double* b, double* x, cudaStream_t s);
  SlabComm& comm_;
  double omega_;
  int coarse_;
  size_t sweeps_;
  std::vector<std::pair<size_t, size_t>> dims_;
  std::vector<std::shared_ptr<DistLevel>> levels_;
  std::vector<Xfer> xfer_;
  std::vector<DevBuf<double>> r_, bc_, xc_;
  std::shared_ptr<Hierarchy> tail_;
  std::vector<size_t> tail_rows_;
  DevBuf<double> tail_b_, tail_full_, tail_x_;
  // captured V-cycle per (b, x) pair (NCCL collectives included)
  struct Entry {
    const double* b;
    double* x;
    cudaGraphExec_t exec;
    unsigned long long kernels;
  };
  std::vector<Entry> graphs_;
  bool use_graphs_ = false;
  cudaStream_t cap_ = nullptr;

 public:
  ~DistHierarchy();
};

struct DistReport {
  size_t iterations = 0;
  bool converged = false;
  double final_rel = 0.0;
};

// gmres (krylov.cpp:34-166) on slab vectors: the control flow of
// KrylovWorkspace::gmres, dots combined across ranks on the device.
class DistGmres {
 public:
  DistGmres(SlabComm& c, std::shared_ptr<DistLevel> a, DistHierarchy* m, size_t restart);
  ~DistGmres();
  DistReport solve(const double* b, double* x, const SolverConfig& cfg, cudaStream_t s);

 private:
  // *slot = sum over ranks (rank order) of <x, y>, square-rooted if asked
  void gdot(const double* x, const double* y, int slot, bool sqrt_out, cudaStream_t s);
  void gsum(int slot, bool sqrt_out, cudaStream_t s);
  void gram_schmidt(size_t i, double* w, int base, cudaStream_t s);
  void fetch(int first, int count, cudaStream_t s);
  void pc(const double* r, double* z, cudaStream_t s);
  SlabComm& comm_;
  std::shared_ptr<DistLevel> a_;
  DistHierarchy* m_;
  size_t n_, rst_;
  std::vector<DevBuf<double>> v_;
  DevBuf<double> t_, r_, z_, w_, trial_;
  DevBuf<double> dsc_, dpart_, dall_, dcoef_;
  DevBuf<const double*> dptr_;
  double* hsc_ = nullptr;  // pinned mirror of dsc_
  Reducer red_;
};

// time_march (driver.cpp:10-69) on y-slabs: the rank's rows of u^m stay on
// its device.
class DistMarch {
 public:
  DistMarch(std::shared_ptr<SlabComm> c, const Problem& p, size_t n1, size_t n2, size_t steps,
            const SolverConfig& cfg, double omega, int coarse, size_t coarse_sweeps,
            size_t agglomerate, bool precond);
  size_t r0() const { return level_->r0; }
  size_t r1() const { return level_->r1; }
  size_t local_size() const { return level_->local_size(); }
  // source_local: the rank's rows of v(., t^{m-1/2}) on the device, or null
  // (BASELINE presets: generated on the device from the counter hash)
  DistReport step(const double* source_local, cudaStream_t s);
  const double* solution() const { return u_.get(); }
  DistLevel& level() { return *level_; }
  DistHierarchy* hierarchy() { return mg_.get(); }
  SlabComm& comm() { return *comm_; }
  size_t steps_taken() const { return m_; }

 private:
  std::shared_ptr<SlabComm> comm_;
  Problem p_;
  Grid g_;
  SolverConfig cfg_;
  std::shared_ptr<DistLevel> level_;
  std::unique_ptr<DistHierarchy> mg_;
  std::unique_ptr<DistGmres> solver_;
  DevBuf<double> u_, b_, x_, src_;
  double scale_ = 0.0;
  size_t m_ = 0;
};

}  // namespace fde_b200

// y-slab multi-GPU time step: transports, slab levels, distributed V-cycle,
// GMRES and march (see dist.cuh).
#include <dlfcn.h>

#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "dist.cuh"
#include "line_conv.cuh"

namespace fde_b200 {

// ------------------------------------------------------------------ partition
std::vector<size_t> split_ranges(size_t n, int parts) {
  std::vector<size_t> o(parts + 1);
  for (int r = 0; r <= parts; ++r) o[r] = n * (size_t)r / (size_t)parts;
  return o;
}

std::vector<size_t> induced_coarse_rows(const std::vector<size_t>& fine_offsets, size_t d2,
                                        bool coarsen_y) {
  if (!coarsen_y) return fine_offsets;
  const long long par = (long long)((d2 + 1) % 2);
  const size_t k2 = coarse_size(d2);
  std::vector<size_t> out;
  for (size_t f : fine_offsets) {  // first coarse row whose centre 2b + 1 - par is >= f
    long long b = 0;
    if (f > 0) {
      const long long t = (long long)f - 1 + par;  // ceil(t / 2), t >= 0
      b = (t + 1) / 2;
    }
    out.push_back(std::min((size_t)b, k2));
  }
  out.back() = k2;
  return out;
}

// ------------------------------------------------------------------ NCCL
namespace {

struct NcclApi {
  using comm_t = void*;
  struct UniqueId {
    char internal[128];
  };
  int (*GetUniqueId)(UniqueId*) = nullptr;
  int (*CommInitRank)(comm_t*, int, UniqueId, int) = nullptr;
  int (*CommDestroy)(comm_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  int (*Send)(const void*, size_t, int, int, comm_t, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, comm_t, cudaStream_t) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, comm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  static constexpr int kFloat64 = 8;  // ncclFloat64

  static NcclApi& get() {
    static NcclApi api = [] {
      NcclApi a;
      void* h = nullptr;
      const char* env = std::getenv("FDE_NCCL_LIB");
      for (const char* name : {env, "libnccl.so.2", "libnccl.so"}) {
        if (!name) continue;
        h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
        if (h) break;
      }
      if (!h) throw RuntimeError("libnccl.so.2 not found (set FDE_NCCL_LIB)");
      auto sym = [&](const char* n) {
        void* p = dlsym(h, n);
        if (!p) throw RuntimeError(std::string("NCCL symbol missing: ") + n);
        return p;
      };
      a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
      a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
      a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
      a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
      a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
      a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
      a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
      a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
      a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
      return a;
    }();
    return api;
  }
  void check(int rc, const char* what) const {
    if (rc != 0)
      throw RuntimeError(std::string("NCCL ") + what + ": " +
                         (GetErrorString ? GetErrorString(rc) : "error"));
  }
};

class NcclComm final : public SlabComm {
 public:
  NcclComm(const void* id128, int rank, int world) : api_(NcclApi::get()) {
    rank_ = rank;
    world_ = world;
    NcclApi::UniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    api_.check(api_.CommInitRank(&comm_, world, id, rank), "ncclCommInitRank");
  }
  ~NcclComm() override {
    if (comm_) api_.CommDestroy(comm_);
  }
  void all_to_all(const double* send, const size_t* scnt, double* recv, const size_t* rcnt,
                  cudaStream_t s) override {
    ++ncoll_;
    api_.check(api_.GroupStart(), "ncclGroupStart");
    size_t so = 0, ro = 0;
    for (int q = 0; q < world_; ++q) {
      if (scnt[q]) api_.check(api_.Send(send + so, scnt[q], NcclApi::kFloat64, q, comm_, s), "ncclSend");
      if (rcnt[q]) api_.check(api_.Recv(recv + ro, rcnt[q], NcclApi::kFloat64, q, comm_, s), "ncclRecv");
      so += scnt[q];
      ro += rcnt[q];
    }
    api_.check(api_.GroupEnd(), "ncclGroupEnd");
  }
  void all_gather(const double* send, double* recv, size_t count, cudaStream_t s) override {
    ++ncoll_;
    api_.check(api_.AllGather(send, recv, count, NcclApi::kFloat64, comm_, s), "ncclAllGather");
  }
  void all_gather_v(const double* send, double* recv, const size_t* counts,
                    cudaStream_t s) override {
    ++ncoll_;
    api_.check(api_.GroupStart(), "ncclGroupStart");
    size_t ro = 0;
    for (int q = 0; q < world_; ++q) {
      if (counts[rank_])
        api_.check(api_.Send(send, counts[rank_], NcclApi::kFloat64, q, comm_, s), "ncclSend");
      if (counts[q])
        api_.check(api_.Recv(recv + ro, counts[q], NcclApi::kFloat64, q, comm_, s), "ncclRecv");
      ro += counts[q];
    }
    api_.check(api_.GroupEnd(), "ncclGroupEnd");
  }
  void halo(const double* send_down, const double* send_up, double* below, double* above,
            size_t width, cudaStream_t s) override {
    if (!send_down && !send_up && !below && !above) return;
    ++ncoll_;
    api_.check(api_.GroupStart(), "ncclGroupStart");
    if (below) api_.check(api_.Recv(below, width, NcclApi::kFloat64, rank_ - 1, comm_, s), "ncclRecv");
    if (above) api_.check(api_.Recv(above, width, NcclApi::kFloat64, rank_ + 1, comm_, s), "ncclRecv");
    if (send_up) api_.check(api_.Send(send_up, width, NcclApi::kFloat64, rank_ + 1, comm_, s), "ncclSend");
    if (send_down)
      api_.check(api_.Send(send_down, width, NcclApi::kFloat64, rank_ - 1, comm_, s), "ncclSend");
    api_.check(api_.GroupEnd(), "ncclGroupEnd");
  }
  bool capturable() const override { return true; }

 private:
  NcclApi& api_;
  NcclApi::comm_t comm_ = nullptr;
};

// ------------------------------------------------------------------ virtual ranks
// P host threads, one device, one stream: a collective is a rendezvous of the
// threads (so every rank's producers are enqueued), device copies enqueued by
// the receivers, and a second rendezvous (so no rank enqueues a kernel that
// overwrites a send buffer ahead of those copies).
struct VirtualGroup {
  explicit VirtualGroup(int p) : P(p), a(p, nullptr), b(p, nullptr), cnt(p, nullptr) {}
  int P;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long gen = 0;
  bool aborted = false;
  std::vector<const double*> a, b;
  std::vector<const size_t*> cnt;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    if (aborted) throw RuntimeError("a virtual rank failed");
    const unsigned long long g = gen;
    if (++arrived == P) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return;
    }
    while (gen == g && !aborted) cv.wait_for(lk, std::chrono::milliseconds(50));
    if (gen == g) throw RuntimeError("a virtual rank failed");
  }
  void abort() {
    std::lock_guard<std::mutex> lk(mu);
    aborted = true;
    cv.notify_all();
  }
};

class VirtualComm final : public SlabComm {
 public:
  VirtualComm(std::shared_ptr<VirtualGroup> g, int rank) : g_(std::move(g)) {
    rank_ = rank;
    world_ = g_->P;
  }
  void all_to_all(const double* send, const size_t* scnt, double* recv, const size_t* rcnt,
                  cudaStream_t s) override {
    ++ncoll_;
    g_->a[rank_] = send;
    g_->cnt[rank_] = scnt;
    g_->barrier();
    size_t ro = 0;
    for (int q = 0; q < world_; ++q) {
      size_t so = 0;
      for (int d = 0; d < rank_; ++d) so += g_->cnt[q][d];
      const size_t c = g_->cnt[q][rank_];
      if (c != rcnt[q]) throw RuntimeError("all-to-all counts disagree");
      if (c) FDE_CUDA(cudaMemcpyAsync(recv + ro, g_->a[q] + so, c * sizeof(double),
                                      cudaMemcpyDeviceToDevice, s));
      ro += c;
    }
    g_->barrier();
  }
  void all_gather(const double* send, double* recv, size_t count, cudaStream_t s) override {
    ++ncoll_;
    g_->a[rank_] = send;
    g_->barrier();
    for (int q = 0; q < world_; ++q)
      if (count) FDE_CUDA(cudaMemcpyAsync(recv + (size_t)q * count, g_->a[q], count * sizeof(double),
                                          cudaMemcpyDeviceToDevice, s));
    g_->barrier();
  }
  void all_gather_v(const double* send, double* recv, const size_t* counts,
                    cudaStream_t s) override {
    ++ncoll_;
    g_->a[rank_] = send;
    g_->barrier();
    size_t ro = 0;
    for (int q = 0; q < world_; ++q) {
      if (counts[q]) FDE_CUDA(cudaMemcpyAsync(recv + ro, g_->a[q], counts[q] * sizeof(double),
                                              cudaMemcpyDeviceToDevice, s));
      ro += counts[q];
    }
    g_->barrier();
  }
  void halo(const double* send_down, const double* send_up, double* below, double* above,
            size_t width, cudaStream_t s) override {
    // every rank takes part (the rendezvous is collective), also with nothing to move
    ++ncoll_;
    g_->a[rank_] = send_down;
    g_->b[rank_] = send_up;
    g_->barrier();
    if (below) {
      if (rank_ == 0 || !g_->b[rank_ - 1]) throw RuntimeError("halo row not offered");
      FDE_CUDA(cudaMemcpyAsync(below, g_->b[rank_ - 1], width * sizeof(double),
                               cudaMemcpyDeviceToDevice, s));
    }
    if (above) {
      if (rank_ + 1 >= world_ || !g_->a[rank_ + 1]) throw RuntimeError("halo row not offered");
      FDE_CUDA(cudaMemcpyAsync(above, g_->a[rank_ + 1], width * sizeof(double),
                               cudaMemcpyDeviceToDevice, s));
    }
    g_->barrier();
  }
  bool capturable() const override { return false; }
  VirtualGroup& group() { return *g_; }

 private:
  std::shared_ptr<VirtualGroup> g_;
};

__global__ void k_ordered_sum(const double* __restrict__ parts, int n, double* __restrict__ out,
                              int sqrt_out) {
  pdl_enter();
  if (threadIdx.x == 0) {
    double acc = parts[0];
    for (int r = 1; r < n; ++r) acc += parts[r];
    *out = sqrt_out ? sqrt(acc) : acc;
  }
}

}  // namespace

void nccl_unique_id(void* id128) {
  NcclApi& api = NcclApi::get();
  NcclApi::UniqueId id;
  api.check(api.GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(id128, &id, sizeof(id));
}
std::shared_ptr<SlabComm> make_nccl_comm(const void* id128, int rank, int world) {
  if (world < 1 || rank < 0 || rank >= world) throw InvalidArgument("bad rank / world size");
  return std::make_shared<NcclComm>(id128, rank, world);
}
std::vector<std::shared_ptr<SlabComm>> make_virtual_comms(int P) {
  if (P < 1 || P > 64) throw InvalidArgument("virtual world size must be 1..64");
  auto g = std::make_shared<VirtualGroup>(P);
  std::vector<std::shared_ptr<SlabComm>> out;
  for (int r = 0; r < P; ++r) out.push_back(std::make_shared<VirtualComm>(g, r));
  return out;
}
void abort_virtual(SlabComm& c) {
  if (auto* v = dynamic_cast<VirtualComm*>(&c)) v->group().abort();
}

// ------------------------------------------------------------------ slab level
DistLevel::DistLevel(SlabComm& c, const Problem& p, size_t nf1, size_t nf2, size_t d1_, size_t d2_,
                     std::vector<size_t> row_offsets, size_t steps, size_t m)
    : comm(c), d1(d1_), d2(d2_), rows(std::move(row_offsets)) {
  const int P = c.world(), r = c.rank();
  if ((int)rows.size() != P + 1 || rows[0] != 0 || rows[P] != d2)
    throw InvalidArgument("row offsets must span the level");
  cols = split_ranges(d1, P);
  r0 = rows[r];
  r1 = rows[r + 1];
  c0 = cols[r];
  c1 = cols[r + 1];
  nr = r1 - r0;
  nc = c1 - c0;
  op_ = std::make_unique<SlabOp>(p, nf1, nf2, d1, d2, steps, m, r0, r1, c0, c1);
  const std::vector<double>& diag = op_->diagonal();
  std::vector<double> inv(diag.size());
  for (size_t i = 0; i < diag.size(); ++i) {
    if (!(diag[i] > 0.0)) throw InvalidArgument("operator diagonal must be strictly positive");
    inv[i] = 1.0 / diag[i];
  }
  dinv.upload(inv.data(), inv.size());
  xTl_.alloc(d1 * nr);
  recv_.alloc(nc * d2);
  xT_.alloc(nc * d2);
  QT_.alloc(nc * d2);
  send2_.alloc(nc * d2);
  recv2_.alloc(d1 * nr);
  Q_.alloc(nr * d1);
  for (int q = 0; q < P; ++q) {
    s1_.push_back((cols[q + 1] - cols[q]) * nr);    // my rows of rank q's columns
    r1_.push_back(nc * (rows[q + 1] - rows[q]));    // rank q's rows of my columns
    s2_.push_back(nc * (rows[q + 1] - rows[q]));
    r2_.push_back((cols[q + 1] - cols[q]) * nr);
  }
  for (size_t v : rows) rows_ll_.push_back((long long)v);
}

void DistLevel::run(const double* x, double* out, double sign, int epi, const EpiArgs& e,
                    cudaStream_t s, const InMap* in) {
  const PdlOff plain;
  const int P = comm.world();
  // [nr][d1] -> [d1][nr]; with an input map x = in(.) is formed (and stored)
  // on the way, as StructuredOp::run_mapped does
  if (nr && in)
    launch_transpose_mapped(*in, const_cast<double*>(x), xTl_.get(), (int)d1, (int)nr, s);
  else if (nr)
    launch_transpose(x, xTl_.get(), (int)d1, (int)nr, s);
  comm.all_to_all(xTl_.get(), s1_.data(), recv_.get(), r1_.data(), s);
  block_permute(recv_.get(), xT_.get(), nc, d2, rows_ll_.data(), P, 0, s);  // -> [nc][d2]
  op_->ypass(xT_.get(), QT_.get(), sign, s);
  block_permute(QT_.get(), send2_.get(), nc, d2, rows_ll_.data(), P, 1, s);
  comm.all_to_all(send2_.get(), s2_.data(), recv2_.get(), r2_.data(), s);
  if (nr) launch_transpose(recv2_.get(), Q_.get(), (int)nr, (int)d1, s);  // [d1][nr] -> [nr][d1]
  op_->xpass(x, Q_.get(), out, sign, epi, e, s);
}

// ------------------------------------------------------------------ V-cycle
namespace {
// Vectors that exchange halo rows are laid out [pad | row below | local rows |
// row above]: the local part starts an even number of doubles into the
// allocation, so it is 16-byte aligned like every other operand of the line
// kernels (their 128-bit path needs all streams to agree modulo 16 bytes).
size_t halo_off(size_t width) { return width + (width & 1); }
size_t halo_len(size_t rows, size_t width) { return halo_off(width) + (rows + 1) * width + 2; }
// which neighbour rows the restriction of fine rows `rows` to coarse rows
// `coarse` needs on rank rk: (row below the slab, row above the slab)
std::pair<bool, bool> restrict_need(const std::vector<size_t>& rows,
                                    const std::vector<size_t>& coarse, size_t a2, int rk) {
  const long long par = (long long)((a2 + 1) % 2);
  const long long lo = (long long)coarse[rk], hi = (long long)coarse[rk + 1];
  if (hi <= lo) return {false, false};
  const long long f_lo = 2 * lo + 1 - par - 1, f_hi = 2 * (hi - 1) + 1 - par + 1;
  return {f_lo < (long long)rows[rk] && f_lo >= 0,
          f_hi >= (long long)rows[rk + 1] && f_hi < (long long)a2};
}
long long floor_div2(long long t) { return t >= 0 ? t / 2 : -((-t + 1) / 2); }
// which coarse neighbour rows the prolongation onto fine rows `rows` needs
std::pair<bool, bool> prolong_need(const std::vector<size_t>& rows,
                                   const std::vector<size_t>& crow, size_t a2, size_t k2, int rk) {
  const long long par = (long long)((a2 + 1) % 2);
  const long long f0 = (long long)rows[rk], f1 = (long long)rows[rk + 1];
  if (f1 <= f0) return {false, false};
  const long long t0 = f0 - 1 + par, t1 = (f1 - 1) - 1 + par;
  const long long lo = (t0 % 2 == 0) ? floor_div2(t0) : floor_div2(t0 - 1);
  const long long hi = (t1 % 2 == 0) ? floor_div2(t1) : floor_div2(t1 + 1);
  return {lo >= 0 && lo < (long long)crow[rk], hi >= (long long)crow[rk + 1] && hi < (long long)k2};
}
}  // namespace

DistHierarchy::DistHierarchy(SlabComm& c, const Problem& p, size_t n1, size_t n2, size_t steps,
                             size_t m, double omega, int coarse, size_t coarse_sweeps,
                             size_t agglomerate, std::shared_ptr<DistLevel> fine)
    : comm_(c), omega_(omega), coarse_(coarse), sweeps_(coarse_sweeps) {
  if (!(omega > 0.0) || coarse < COARSE_LU || coarse > COARSE_NONE)
    throw InvalidArgument("invalid multigrid configuration");
  const Grid g(p, n1, n2, steps);
  {
    // the level plan of the full fine operator (multigrid.cpp:116-158); the
    // operator itself is dropped again
    auto full = assemble_step_operator(p, g, m);
    dims_ = plan_level_dims(n1, n2, anisotropy_ratio(*full, p.alpha, p.beta), p.alpha, p.beta);
  }
  const size_t L = dims_.size();
  const int P = c.world();
  levels_.push_back(std::move(fine));
  std::vector<size_t> offsets = levels_[0]->rows;
  size_t ls = 1;
  while (ls < L) {
    const size_t l1 = dims_[ls].first, l2 = dims_[ls].second, pd2 = dims_[ls - 1].second;
    std::vector<size_t> nxt = induced_coarse_rows(offsets, pd2, l2 < pd2);
    size_t min_rows = l2;
    for (int r = 0; r < P; ++r) min_rows = std::min(min_rows, nxt[r + 1] - nxt[r]);
    if (l1 * l2 <= agglomerate || min_rows < 2) break;
    levels_.push_back(std::make_shared<DistLevel>(c, p, n1, n2, l1, l2, nxt, steps, m));
    offsets = std::move(nxt);
    ++ls;
  }
  for (size_t l = 0; l + 1 < L; ++l)
    xfer_.push_back(make_xfer((int)dims_[l].first, (int)dims_[l].second,
                              dims_[l + 1].first < dims_[l].first,
                              dims_[l + 1].second < dims_[l].second));
  // residuals and coarse iterates carry one halo row on each side
  r_.resize(ls);
  bc_.resize(ls);
  xc_.resize(ls);
  for (size_t l = 0; l < ls; ++l) {
    const DistLevel& lv = *levels_[l];
    r_[l].alloc(halo_len(lv.nr, lv.d1));
    if (l) {
      bc_[l].alloc(lv.local_size() + 1);
      xc_[l].alloc(halo_len(lv.nr, lv.d1));
    }
  }
  if (ls < L) {
    std::vector<LevelOp> tl;
    std::vector<std::pair<size_t, size_t>> td(dims_.begin() + ls, dims_.end());
    for (const auto& d : td) {
      const Grid lg(p, d.first, d.second, steps);
      LevelOp lev;
      lev.sop = assemble_step_operator(p, lg, m);
      lev.sop->scale(std::pow(g.hx / lg.hx, p.alpha));  // multigrid.cpp:421-427
      tl.push_back(std::move(lev));
    }
    tail_ = std::make_shared<Hierarchy>(std::move(tl), td, MODE_GEOMETRIC, omega, coarse,
                                        coarse_sweeps);
    const DistLevel& last = *levels_.back();
    tail_rows_ = induced_coarse_rows(last.rows, last.d2, xfer_[ls - 1].cy != 0);
    const size_t k1 = dims_[ls].first, k2 = dims_[ls].second;
    tail_b_.alloc((tail_rows_[c.rank() + 1] - tail_rows_[c.rank()]) * k1 + 1);
    tail_full_.alloc(k1 * k2);
    tail_x_.alloc(k1 * k2);
  } else if (coarse == COARSE_LU) {
    throw InvalidArgument("LU coarsest solve on a slab level: raise `agglomerate`");
  }
  if (const char* e = std::getenv("FDE_DIST_GRAPH")) use_graphs_ = e[0] == '1';
  else use_graphs_ = c.capturable();
  if (!c.capturable()) use_graphs_ = false;
}

DistHierarchy::~DistHierarchy() {
  for (Entry& e : graphs_) cudaGraphExecDestroy(e.exec);
  if (cap_) cudaStreamDestroy(cap_);
}

void DistHierarchy::sweep(size_t l, const double* b, double* x, cudaStream_t s) {
  DistLevel& lv = *levels_[l];
  EpiArgs e;
  e.b = b;
  e.dinv = lv.dinv.get();
  e.omega = omega_;
  lv.run(x, x, 1.0, EPI_JACOBI, e, s);  // x += omega dinv (b - A x), multigrid.cpp:364-383
}

void DistHierarchy::restrict_to(size_t l, const double* r_local, double* out, size_t c_lo,
                                size_t c_hi, cudaStream_t s) {
  // r_local sits inside a halo-padded buffer: the row below starts d1 before it
  DistLevel& lv = *levels_[l];
  const Xfer& t = xfer_[l];
  const double* r_pad = r_local - lv.d1;
  if (!t.cy) {
    xfer_restrict_rows(t, r_local, (int)lv.r0, out, (int)c_lo, (int)(c_hi - c_lo), 0.5, s);
    return;
  }
  const int P = comm_.world(), rk = comm_.rank();
  const std::vector<size_t> coarse = induced_coarse_rows(lv.rows, lv.d2, true);
  const auto mine = restrict_need(lv.rows, coarse, lv.d2, rk);
  const bool up_wants = rk + 1 < P && restrict_need(lv.rows, coarse, lv.d2, rk + 1).first;
  const bool down_wants = rk > 0 && restrict_need(lv.rows, coarse, lv.d2, rk - 1).second;
  double* pad = const_cast<double*>(r_pad);
  comm_.halo(down_wants && lv.nr ? r_local : nullptr,
             up_wants && lv.nr ? r_local + (lv.nr - 1) * lv.d1 : nullptr,
             mine.first ? pad : nullptr, mine.second ? pad + (lv.nr + 1) * lv.d1 : nullptr, lv.d1,
             s);
  if (mine.first)
    xfer_restrict_rows(t, r_pad, (int)lv.r0 - 1, out, (int)c_lo, (int)(c_hi - c_lo), 0.5, s);
  else
    xfer_restrict_rows(t, r_local, (int)lv.r0, out, (int)c_lo, (int)(c_hi - c_lo), 0.5, s);
}

void DistHierarchy::prolong_add(size_t l, const double* xc_local, double* x, cudaStream_t s) {
  DistLevel& lv = *levels_[l];
  DistLevel& nx = *levels_[l + 1];
  const Xfer& t = xfer_[l];
  const double* xc_pad = xc_local - nx.d1;
  if (!t.cy) {
    xfer_prolong_rows(t, xc_local, (int)nx.r0, x, (int)lv.r0, (int)lv.nr, true, s);
    return;
  }
  const int P = comm_.world(), rk = comm_.rank();
  const auto mine = prolong_need(lv.rows, nx.rows, lv.d2, nx.d2, rk);
  const bool up_wants = rk + 1 < P && prolong_need(lv.rows, nx.rows, lv.d2, nx.d2, rk + 1).first;
  const bool down_wants = rk > 0 && prolong_need(lv.rows, nx.rows, lv.d2, nx.d2, rk - 1).second;
  double* pad = const_cast<double*>(xc_pad);
  comm_.halo(down_wants && nx.nr ? xc_local : nullptr,
             up_wants && nx.nr ? xc_local + (nx.nr - 1) * nx.d1 : nullptr,
             mine.first ? pad : nullptr, mine.second ? pad + (nx.nr + 1) * nx.d1 : nullptr, nx.d1,
             s);
  if (mine.first)
    xfer_prolong_rows(t, xc_pad, (int)nx.r0 - 1, x, (int)lv.r0, (int)lv.nr, true, s);
  else
    xfer_prolong_rows(t, xc_local, (int)nx.r0, x, (int)lv.r0, (int)lv.nr, true, s);
}

void DistHierarchy::cycle(size_t l, const double* b, double* x, bool zero, cudaStream_t s) {
  DistLevel& lv = *levels_[l];
  const size_t n = lv.local_size();
  const bool last_slab = l + 1 == levels_.size();
  auto presmooth = [&] {
    if (zero) vec_diag_scale(n, omega_, lv.dinv.get(), b, x, s);  // multigrid.cpp:355-356
    else sweep(l, b, x, s);
  };
  if (last_slab && !tail_) {  // the coarsest level is a slab level
    if (coarse_ == COARSE_SWEEPS) {
      presmooth();
      for (size_t k = 1; k < sweeps_; ++k) sweep(l, b, x, s);
    } else if (zero) {
      FDE_CUDA(cudaMemsetAsync(x, 0, n * sizeof(double), s));  // CoarseSolve::none
    }
    return;
  }
  double* r_local = r_[l].get() + halo_off(lv.d1);
  EpiArgs e;
  e.b = b;
  if (zero) {
    // x = omega dinv b rides on the residual's local transpose (multigrid.cpp:355-356)
    InMap zin{};
    zin.kind = 1;
    zin.a = b;
    zin.d = lv.dinv.get();
    zin.w = omega_;
    zin.ld = (int)lv.d1;
    lv.run(x, r_local, 1.0, EPI_RESID, e, s, &zin);  // x, r = b - A x
  } else {
    presmooth();
    lv.run(x, r_local, 1.0, EPI_RESID, e, s);  // r = b - A x
  }
  if (last_slab) {
    const int rk = comm_.rank(), P = comm_.world();
    const size_t k1 = dims_[l + 1].first;
    restrict_to(l, r_local, tail_b_.get(), tail_rows_[rk], tail_rows_[rk + 1], s);
    std::vector<size_t> counts(P);
    for (int q = 0; q < P; ++q) counts[q] = (tail_rows_[q + 1] - tail_rows_[q]) * k1;
    comm_.all_gather_v(tail_b_.get(), tail_full_.get(), counts.data(), s);
    if (tail_->coarse() == COARSE_NONE) tail_x_.zero(s);
    tail_->vcycle(tail_full_.get(), tail_x_.get(), true, s);
    xfer_prolong_rows(xfer_[l], tail_x_.get(), 0, x, (int)lv.r0, (int)lv.nr, true, s);
  } else {
    DistLevel& nx = *levels_[l + 1];
    restrict_to(l, r_local, bc_[l + 1].get(), nx.r0, nx.r1, s);
    double* xc_local = xc_[l + 1].get() + halo_off(nx.d1);
    cycle(l + 1, bc_[l + 1].get(), xc_local, true, s);
    prolong_add(l, xc_local, x, s);
  }
  sweep(l, b, x, s);  // post-smoothing
}

void DistHierarchy::record(const double* b, double* x, cudaStream_t s) { cycle(0, b, x, true, s); }

void DistHierarchy::vcycle(const double* b, double* x, cudaStream_t s) {
  const PdlOff plain;
  if (!use_graphs_) {
    record(b, x, s);
    return;
  }
  for (const Entry& e : graphs_)
    if (e.b == b && e.x == x) {
      FDE_CUDA(cudaGraphLaunch(e.exec, s));
      g_kernel_launches.fetch_add(e.kernels, std::memory_order_relaxed);
      return;
    }
  if (!cap_) FDE_CUDA(cudaStreamCreateWithFlags(&cap_, cudaStreamNonBlocking));
  cudaGraph_t g = nullptr;
  const unsigned long long before = g_kernel_launches.load();
  FDE_CUDA(cudaStreamBeginCapture(cap_, cudaStreamCaptureModeRelaxed));
  try {
    record(b, x, cap_);
  } catch (...) {
    cudaStreamEndCapture(cap_, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  FDE_CUDA(cudaStreamEndCapture(cap_, &g));
  cudaGraphExec_t exec = nullptr;
  const cudaError_t err = cudaGraphInstantiate(&exec, g, 0);
  cudaGraphDestroy(g);
  FDE_CUDA(err);
  graphs_.push_back(Entry{b, x, exec, g_kernel_launches.load() - before});
  FDE_CUDA(cudaGraphLaunch(exec, s));
}

// ------------------------------------------------------------------ GMRES
namespace {
std::vector<double> back_sub(const std::vector<double>& h, size_t ld, const std::vector<double>& g,
                             size_t k) {  // krylov.cpp:19-30
  std::vector<double> y(k, 0.0);
  for (size_t i = k; i-- > 0;) {
    double v = g[i];
    for (size_t j = i + 1; j < k; ++j) v -= h[j * ld + i] * y[j];
    y[i] = h[i * ld + i] != 0.0 ? v / h[i * ld + i] : 0.0;
  }
  return y;
}
}  // namespace

// device scalar slots: [0] ||w|| before Gram-Schmidt, [1 + k] h_k (k <= i),
// [2 + i] ||w|| after; a second block of the same size for the second
// Gram-Schmidt pass; one slot for stand-alone norms
DistGmres::DistGmres(SlabComm& c, std::shared_ptr<DistLevel> a, DistHierarchy* m, size_t restart)
    : comm_(c), a_(std::move(a)), m_(m), n_(a_->local_size()), rst_(restart) {
  if (restart == 0) throw InvalidArgument("invalid solver configuration");
  v_.resize(rst_ + 1);
  std::vector<const double*> ptrs(rst_ + 1);
  for (size_t k = 0; k <= rst_; ++k) {
    v_[k].alloc(n_ + 1);
    ptrs[k] = v_[k].get();
  }
  dptr_.upload(ptrs.data(), ptrs.size());
  t_.alloc(n_ + 1);
  r_.alloc(n_ + 1);
  z_.alloc(n_ + 1);
  w_.alloc(n_ + 1);
  trial_.alloc(n_ + 1);
  const size_t slots = 2 * (rst_ + 3) + 1;
  dsc_.alloc(slots);
  dsc_.zero();
  dpart_.alloc(1);
  dall_.alloc(c.world());
  dcoef_.alloc(rst_ + 1);
  FDE_CUDA(cudaMallocHost(&hsc_, (slots + rst_ + 1) * sizeof(double)));
}
DistGmres::~DistGmres() {
  if (hsc_) cudaFreeHost(hsc_);
}

// this rank's partial in dpart_ -> the rank-ordered global sum in slot
void DistGmres::gsum(int slot, bool sqrt_out, cudaStream_t s) {
  comm_.all_gather(dpart_.get(), dall_.get(), 1, s);
  launch_k(k_ordered_sum, 1, 32, 0, s, (const double*)dall_.get(), comm_.world(),
           dsc_.get() + slot, sqrt_out ? 1 : 0);
  FDE_LAUNCH_CHECK();
}
void DistGmres::gdot(const double* x, const double* y, int slot, bool sqrt_out, cudaStream_t s) {
  if (n_) red_.dot(n_, x, y, dpart_.get(), s, false);
  else dpart_.zero(s);
  gsum(slot, sqrt_out, s);
}
// One modified Gram-Schmidt sweep over v_0 .. v_i with the coefficients in
// slots base + 1 + k and the final norm in base + 2 + i (krylov.cpp:92-97):
// each subtraction w -= h_k v_k is fused with the next projection <v_{k+1}, w>
// (the last with ||w||^2) -- one pass over w per basis vector instead of two
void DistGmres::gram_schmidt(size_t i, double* w, int base, cudaStream_t s) {
  gdot(v_[0].get(), w, base + 1, false, s);
  for (size_t k = 0; k <= i; ++k) {
    if (n_)
      red_.mgs(n_, w, v_[k].get(), dsc_.get() + base + 1 + k, k < i ? v_[k + 1].get() : w,
               dpart_.get(), false, s);
    else
      dpart_.zero(s);
    gsum(base + 2 + (int)k, k == i, s);
  }
}

void DistGmres::fetch(int first, int count, cudaStream_t s) {
  FDE_CUDA(cudaMemcpyAsync(hsc_ + first, dsc_.get() + first, count * sizeof(double),
                           cudaMemcpyDeviceToHost, s));
  FDE_CUDA(cudaStreamSynchronize(s));
}

void DistGmres::pc(const double* r, double* z, cudaStream_t s) {
  if (!m_) FDE_CUDA(cudaMemcpyAsync(z, r, n_ * sizeof(double), cudaMemcpyDeviceToDevice, s));
  else m_->vcycle(r, z, s);
}

DistReport DistGmres::solve(const double* b, double* x, const SolverConfig& cfg, cudaStream_t s) {
  if (cfg.restart != rst_ || cfg.max_outer == 0 || !(cfg.tol > 0.0))
    throw InvalidArgument("invalid solver configuration");
  const PdlOff plain;
  const int blk = (int)rst_ + 3, NRM = 2 * blk;
  DistReport rep;
  FDE_CUDA(cudaMemsetAsync(x, 0, n_ * sizeof(double), s));
  pc(b, z_.get(), s);
  gdot(z_.get(), z_.get(), NRM, true, s);
  fetch(NRM, 1, s);
  const double norm_b = hsc_[NRM];
  if (norm_b == 0.0) {
    rep.converged = true;
    return rep;
  }
  const size_t ld = rst_ + 1;
  std::vector<double> h(ld * rst_, 0.0), cs(rst_, 0.0), sn(rst_, 0.0), g(ld, 0.0);
  double* xbuf[2] = {x, trial_.get()};
  size_t xver = 0, zver = 0;
  double zbeta = norm_b;
  // ||M^-1 (b - A x)|| of the current iterate; the zero start and an accepted
  // verification are reused bit for bit instead of recomputed
  auto residual_z = [&]() {
    if (zver == xver) return zbeta;
    EpiArgs e;
    e.b = b;
    a_->run(xbuf[0], r_.get(), 1.0, EPI_RESID, e, s);
    pc(r_.get(), z_.get(), s);
    gdot(z_.get(), z_.get(), NRM, true, s);
    fetch(NRM, 1, s);
    zbeta = hsc_[NRM];
    zver = xver;
    return zbeta;
  };
  double* hcoef = hsc_ + 2 * blk + 1;
  auto lincomb = [&](double* dst, const double* src, const std::vector<double>& y) {
    for (size_t k = 0; k < y.size(); ++k) hcoef[k] = y[k];
    FDE_CUDA(cudaMemcpyAsync(dcoef_.get(), hcoef, y.size() * sizeof(double),
                             cudaMemcpyHostToDevice, s));
    vec_lincomb(n_, src, dptr_.get(), dcoef_.get(), (int)y.size(), dst, s);
    FDE_CUDA(cudaStreamSynchronize(s));  // hcoef is reused
  };
  bool converged = false;
  for (size_t outer = 0; outer < cfg.max_outer && !converged; ++outer) {
    const double beta = residual_z();
    const double rel0 = beta / norm_b;
    if (rel0 <= cfg.tol) {
      converged = true;
      break;
    }
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    vec_copy_scale(n_, 1.0 / beta, z_.get(), v_[0].get(), s);
    size_t spanned = 0;
    bool done = false;
    for (size_t i = 0; i < rst_ && !done; ++i) {
      a_->run(v_[i].get(), t_.get(), 1.0, EPI_STORE, EpiArgs{}, s);
      pc(t_.get(), w_.get(), s);
      double* w = w_.get();
      gdot(w, w, 0, true, s);  // ||w||
      gram_schmidt(i, w, 0, s);
      vec_scale_inv_dev(n_, dsc_.get() + 2 + i, w, v_[i + 1].get(), s);
      fetch(0, (int)i + 3, s);  // the step's one host read
      const double norm0 = hsc_[0];
      for (size_t k = 0; k <= i; ++k) h[i * ld + k] = hsc_[1 + k];
      double nrmw = hsc_[2 + i];
      if (nrmw < 1e-8 * norm0) {  // second pass, krylov.cpp:98-104
        gram_schmidt(i, w, blk, s);
        vec_scale_inv_dev(n_, dsc_.get() + blk + 2 + i, w, v_[i + 1].get(), s);
        fetch(blk, (int)i + 3, s);
        for (size_t k = 0; k <= i; ++k) h[i * ld + k] += hsc_[blk + 1 + k];
        nrmw = hsc_[blk + 2 + i];
      }
      const double hip = nrmw;
      const bool happy = hip <= 1e-14 * (norm0 > 0.0 ? norm0 : 1.0);
      for (size_t k = 0; k < i; ++k) {  // previous rotations, krylov.cpp:108-113
        const double tmp = cs[k] * h[i * ld + k] + sn[k] * h[i * ld + k + 1];
        h[i * ld + k + 1] = -sn[k] * h[i * ld + k] + cs[k] * h[i * ld + k + 1];
        h[i * ld + k] = tmp;
      }
      const double denom = std::hypot(h[i * ld + i], hip);
      cs[i] = denom > 0.0 ? h[i * ld + i] / denom : 1.0;
      sn[i] = denom > 0.0 ? hip / denom : 0.0;
      h[i * ld + i] = denom;
      g[i + 1] = -sn[i] * g[i];
      g[i] = cs[i] * g[i];
      ++rep.iterations;
      spanned = i + 1;
      const double est = std::fabs(g[i + 1]) / norm_b;
      if (est <= cfg.tol || happy) {
        lincomb(xbuf[1], xbuf[0], back_sub(h, ld, g, spanned));
        std::swap(xbuf[0], xbuf[1]);
        ++xver;
        if (residual_z() / norm_b <= cfg.tol) {
          converged = true;
          done = true;
        } else if (happy) {
          done = true;
        } else {
          std::swap(xbuf[0], xbuf[1]);  // estimate not confirmed: keep iterating
          ++xver;
        }
      }
    }
    if (!converged && !done) {
      lincomb(xbuf[0], xbuf[0], back_sub(h, ld, g, spanned));
      ++xver;
    }
  }
  const double final_rel = residual_z() / norm_b;
  if (final_rel <= cfg.tol) converged = true;
  rep.final_rel = final_rel;
  rep.converged = converged;
  if (xbuf[0] != x)
    FDE_CUDA(cudaMemcpyAsync(x, xbuf[0], n_ * sizeof(double), cudaMemcpyDeviceToDevice, s));
  return rep;
}

// ------------------------------------------------------------------ march
DistMarch::DistMarch(std::shared_ptr<SlabComm> c, const Problem& p, size_t n1, size_t n2,
                     size_t steps, const SolverConfig& cfg, double omega, int coarse,
                     size_t coarse_sweeps, size_t agglomerate, bool precond)
    : comm_(std::move(c)), p_(p), g_(p, n1, n2, steps), cfg_(cfg) {
  if (p.time_dependent_coeffs)
    // the operator and the hierarchy are built once (at m = 1); a
    // time-dependent problem needs the t^{m-1} operator for the rhs and the
    // step-m operator and V-cycle for the solve (driver.cpp:37-51)
    throw InvalidArgument("the y-slab march supports time-independent coefficients only");
  if ((size_t)comm_->world() > n2 / 2) throw InvalidArgument("too many ranks for this grid");
  level_ = std::make_shared<DistLevel>(*comm_, p, n1, n2, n1, n2, split_ranges(n2, comm_->world()),
                                       steps, 1);
  if (precond)
    mg_ = std::make_unique<DistHierarchy>(*comm_, p, n1, n2, steps, 1, omega, coarse,
                                          coarse_sweeps, agglomerate, level_);
  solver_ = std::make_unique<DistGmres>(*comm_, level_, mg_.get(), cfg.restart);
  const std::vector<double> u0 = sample_initial(p, g_);
  const size_t nl = level_->local_size();
  u_.upload(u0.data() + level_->r0 * n1, nl);
  b_.alloc(nl + 1);
  x_.alloc(nl + 1);
  scale_ = 2.0 * std::pow(g_.hx, p.alpha);  // problem.cpp:82
}

DistReport DistMarch::step(const double* source_local, cudaStream_t s) {
  const PdlOff plain;
  ++m_;
  const size_t n1 = g_.n1;
  if (!source_local) {
    if (src_.size() != g_.size()) src_.alloc(g_.size());
    if (p_.preset && !(p_.preset >= 101)) {
      generate_source_device(p_, g_, m_, src_.get(), s);
    } else {
      std::vector<double> v(g_.size());
      sample_source(p_, g_, m_, v.data());
      FDE_CUDA(cudaMemcpyAsync(src_.get(), v.data(), v.size() * sizeof(double),
                               cudaMemcpyHostToDevice, s));
      FDE_CUDA(cudaStreamSynchronize(s));
    }
    source_local = src_.get() + level_->r0 * n1;
  }
  EpiArgs e;
  e.src = source_local;
  e.src_scale = scale_;
  level_->run(u_.get(), b_.get(), -1.0, EPI_RHS, e, s);  // problem.cpp:73-89
  const DistReport rep = solver_->solve(b_.get(), x_.get(), cfg_, s);
  std::swap(u_, x_);
  return rep;
}

}  // namespace fde_b200

// Host side of the hot path: buffers, launch geometry, and the projected-gradient
// driver that restates ndconv::deconv_pg (solvers.hpp:155-238) with device-resident
// tensors.  See ndc_plan.h for the contract and DESIGN.md for the data layout.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <initializer_list>
#include <string>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <functional>
#include <fcntl.h>
#include <unistd.h>

#include <cstdio>

#include "ndc_io.h"
#include "ndc_plan.h"
#include "ndc_sim.h"

namespace ndc {

namespace {
void* small_pinned_get(size_t bytes);
void small_pinned_put(size_t bytes, void* p);
}  // namespace

namespace {
// Device scalar slots (doubles), per image unless noted.
enum Slot { kF = 0, kKKT = 1, kCHG = 2, kAUX = 3, kNumSlots = 4 };
constexpr int kMaxPowerIters = 4096;
constexpr int kElemBlocks = 148 * 4;  // elementwise kernels: blocks per image

double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

long long cdiv(long long a, long long b) { return (a + b - 1) / b; }
}  // namespace

// Guard-band mode (NDC_GUARD_BANDS=1; tests/test_gpu_guards.py): every plan allocation
// gets kGuard bytes of a fill pattern on both sides, checked when the plan checks or
// frees it -- an out-of-bounds device write into a neighbour's memory shows up as a
// changed guard byte (compute-sanitizer is not available on the GPU pool).
namespace {
constexpr size_t kGuard = size_t(1) << 20;
constexpr unsigned char kGuardByte = 0xA5;
bool guard_mode() {
  static const bool on = [] {
    const char* e = std::getenv("NDC_GUARD_BANDS");
    return e != nullptr && std::atoi(e) != 0;
  }();
  return on;
}
std::atomic<unsigned long long> g_guard_violations{0};
}  // namespace

void fail(int code, const std::string& msg) { throw Error{code, msg}; }

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver ? NDC_ERR_NO_DEVICE : NDC_ERR_CUDA,
         std::string(what) + ": " + cudaGetErrorString(e));
  }
}

Vol Vol::make(int z, int y, int x, int r0, int c0) {
  Vol v;
  v.ez = z;
  v.ey = y;
  v.ex = x;
  v.r0 = r0;
  v.c0 = c0;
  // every output tile (kTileX wide) stays inside its row
  v.pitch = cdiv(c0 + cdiv(x, kTileX) * kTileX, 32) * 32;
  v.plane = v.pitch * (r0 + y);
  v.image = v.plane * z;
  v.origin = static_cast<long long>(r0) * v.pitch + c0;
  return v;
}

Plan::Plan(int device, size_t batch, int ndim, const size_t* x_ext, const size_t* k_ext,
           const double* h, std::unique_ptr<Transport> comm)
    : device_(device), B_(batch), ndim_(ndim), comm_(std::move(comm)) {
  if (ndim < 1) fail(NDC_ERR_SHAPE, "Shape: need at least one dimension");
  if (ndim > kMaxDims)
    fail(NDC_ERR_UNSUPPORTED, "ndconv_b200: at most " + std::to_string(kMaxDims) + " dimensions, got " +
                                  std::to_string(ndim));
  if (batch == 0) fail(NDC_ERR_ARGUMENT, "ndconv_b200: batch must be positive");
  size_t count = 1;
  for (int i = 0; i < ndim; ++i) {
    if (x_ext[i] == 0) fail(NDC_ERR_SHAPE, "Shape: extents must be positive");
    if (k_ext[i] == 0) fail(NDC_ERR_SHAPE, "Shape: extents must be positive");
    if (k_ext[i] % 2 == 0) fail(NDC_ERR_SHAPE, "Kernel: extents must be odd");
    count *= k_ext[i];
  }
  for (size_t i = 0; i < count; ++i)
    if (!std::isfinite(h[i])) fail(NDC_ERR_NUMERIC, "Kernel: values must be finite");
  uext_x_.assign(x_ext, x_ext + ndim);
  uext_k_.assign(k_ext, k_ext + ndim);
  std::vector<double> hm;  // the kernel on the merged plane axis (ndim > 3)
  if (ndim <= 3) {
    const int lead = 3 - ndim;
    for (int i = 0; i < ndim; ++i) {
      xext_[lead + i] = x_ext[i];
      kext_[lead + i] = k_ext[i];
    }
  } else {
    // More than 3 dimensions (the reference recurses over any ndim, convolution.hpp:55-74):
    // dims 0 .. ndim-3 merge into ONE plane axis with the observation's strides, y
    // plane index Z = sum_i z_i S_i (S_{L-1} = 1, S_i = S_{i+1} Y_{i+1}, Y_i = m_i + k_i - 1).
    // x sits at the same indices (zero planes where some z_i >= m_i) and the kernel at
    // J = sum_i j_i S_i (zero slices elsewhere), so a full / valid correlation along the
    // merged axis is exactly the n-d one: Z = z + j never carries between dims because
    // z_i + j_i < Y_i.  The forward pass skips the all-zero tap slices (see build_chunks),
    // the adjoint computes only x's real planes (xruns_), so the zero planes stay zero.
    if (batch != 1) fail(NDC_ERR_UNSUPPORTED, "ndconv_b200: batches of tensors with more than 3 dimensions");
    if (comm_) fail(NDC_ERR_UNSUPPORTED, "ndconv_b200: z-slab sharding handles 1- to 3-d tensors");
    merged_ = true;
    const int L = ndim - 2;
    std::vector<long long> Y(L), S(L);
    for (int i = 0; i < L; ++i) Y[i] = static_cast<long long>(x_ext[i] + k_ext[i] - 1);
    S[L - 1] = 1;
    for (int i = L - 2; i >= 0; --i) S[i] = S[i + 1] * Y[i + 1];
    const long long P = S[0] * Y[0];
    long long KZm = 1;
    for (int i = 0; i < L; ++i) KZm += static_cast<long long>(k_ext[i] - 1) * S[i];
    const long long kyx = static_cast<long long>(k_ext[ndim - 2]) * k_ext[ndim - 1];
    if (P > (1LL << 30) || KZm * kyx > (1LL << 28))
      fail(NDC_ERR_UNSUPPORTED, "ndconv_b200: merged leading dimensions too large");
    xext_[0] = static_cast<size_t>(P);
    xext_[1] = x_ext[ndim - 2];
    xext_[2] = x_ext[ndim - 1];
    kext_[0] = static_cast<size_t>(KZm);
    kext_[1] = k_ext[ndim - 2];
    kext_[2] = k_ext[ndim - 1];
    hm.assign(static_cast<size_t>(KZm * kyx), 0.0);
    for (size_t f = 0; f < count; ++f) {
      size_t rem = f / static_cast<size_t>(kyx);
      long long J = 0;
      for (int i = L - 1; i >= 0; --i) {
        J += static_cast<long long>(rem % k_ext[i]) * S[i];
        rem /= k_ext[i];
      }
      hm[static_cast<size_t>(J * kyx) + f % static_cast<size_t>(kyx)] = h[f];
    }
    // x's real planes: one run of m_{L-1} planes per leading index (z_0 .. z_{L-2})
    std::vector<size_t> idx(L - 1, 0);
    for (;;) {
      long long start = 0;
      for (int i = 0; i < L - 1; ++i) start += static_cast<long long>(idx[i]) * S[i];
      xruns_.push_back({static_cast<int>(start), static_cast<int>(x_ext[L - 1])});
      int i = L - 2;
      for (; i >= 0; --i) {
        if (++idx[i] < x_ext[i]) break;
        idx[i] = 0;
      }
      if (i < 0) break;
    }
    ny_user_planes_ = static_cast<int>(P);
  }
  mz_ = static_cast<int>(xext_[0]);
  my_ = static_cast<int>(xext_[1]);
  mx_ = static_cast<int>(xext_[2]);
  KZ_ = static_cast<int>(kext_[0]);
  KY_ = static_cast<int>(kext_[1]);
  KX_ = static_cast<int>(kext_[2]);
  pz_ = (KZ_ - 1) / 2;
  py_ = (KY_ - 1) / 2;
  px_ = (KX_ - 1) / 2;
  if (static_cast<long long>(my_) + 2 * py_ > (1 << 30) || static_cast<long long>(mx_) + 2 * px_ > (1 << 30))
    fail(NDC_ERR_UNSUPPORTED, "ndconv_b200: extent too large");
  // Kernels of any odd size: a launch carries a tap block of at most kMaxKX columns x
  // kcy_ rows x (as many z-slices as fit kTapCap); larger PSFs run as several launches
  // accumulated through a scratch volume (see correlate()).  Column chunks start at
  // multiples of 32 (keeps the TMA tile origin 16-byte aligned) and are padded with zero
  // taps to an instantiated odd width.
  kcx_ = KX_ <= kMaxKX ? KX_ : kMaxKX;
  // Two output rows per thread (tile height 128) halves the per-row tap loads and loop
  // overhead; used for single-plane (2-D / batched) problems whose 128+KY-1 staged rows
  // fit one TMA box.  For 3-D volumes two 128-row plane stages must also leave room for two
  // CTAs per SM (configs 3 and 4); otherwise see the one-stage rule below (config 5).
  stages_ = (KZ_ > 1) ? 2 : 1;
  {
    const long long pitch2 = std::max(shared_pitch_for(kcx_, 0), shared_pitch_for(kcx_, 2));
    const long long stage2 = static_cast<long long>(2 * kTileY + KY_ - 1) * pitch2 * 4;
    const bool fits = 2 * kTileY + KY_ - 1 <= kMaxRows;
    // two CTAs per SM: staged-epilogue kernels (KX <= kStagedMaxKX) also carry a 16 KB
    // staging buffer; the direct-epilogue ones do not (config 3 runs RY = 2 since then:
    // adjoint +2 %, forward unchanged)
    const long long budget = (kcx_ <= kStagedMaxKX ? 90 : 110) * 1024LL;
    ry_ = (fits && (KZ_ == 1 || stages_ * stage2 <= budget)) ? 2 : 1;
    // small PSFs are HBM-bound: 64-row tiles at 5 CTAs / SM keep more loads in flight
    if (KX_ <= kSmallMaxKX) ry_ = 1;
    // Wide 3-D PSFs whose two 128-row stages do not fit: ONE 128-row stage per CTA and three
    // CTAs / SM (the scalar direct-epilogue kernels of KX >= 23 run at 80 registers) beat
    // 64-row tiles on a two-stage ring at two CTAs / SM -- two rows per lane share every tap
    // load, and a CTA's wait for its next plane hides behind the other two.  Config 5
    // (65 x 33 x 33): forward +3.0 %, adjoint +1.4 % (profiles/r02i_c5_tiles.txt).
    if (KZ_ > 1 && ry_ == 1 && fits && kcx_ >= 23 && 3 * (stage2 + 1024) <= 225 * 1024LL) {
      ry_ = 2;
      stages_ = 1;
    }
  }
  kcy_ = std::min(KY_, kMaxRows - kTileY * ry_ + 1);  // staged rows 64*ry + kcy - 1 <= TMA box limit

  if (merged_)
    h64_ = std::move(hm);
  else
    h64_.assign(h, h + count);
  set_taps(1.0);
  kernel_all_zero_ = true;
  for (size_t i = 0; i < count; ++i)
    if (h[i] != 0.0) kernel_all_zero_ = false;

  // z-slab geometry: rank r owns x planes [xa, xb) and y planes
  // [xa+pz, xb+pz) (the first rank also [0, pz), the last up to mz+2pz).
  if (comm_) {
    rank_ = comm_->rank();
    world_ = comm_->world();
    if (B_ != 1) fail(NDC_ERR_ARGUMENT, "ndconv_b200: sharded plans hold one image");
  }
  size_t a, b, ya, yb;
  ndc_slab_range(static_cast<size_t>(mz_), static_cast<size_t>(pz_), rank_, world_, &a, &b, &ya, &yb);
  xa_ = static_cast<int>(a);
  xb_ = static_cast<int>(b);
  xa_n_ = xb_ - xa_;
  ya_ = static_cast<int>(ya);
  yb_ = static_cast<int>(yb);
  if (world_ > 1 && xa_n_ < pz_)
    fail(NDC_ERR_UNSUPPORTED, "ndconv_b200: z-slab of " + std::to_string(xa_n_) +
                                  " planes is thinner than the halo (" + std::to_string(pz_) + ")");
  xlo_ = std::max(0, xa_ - pz_);
  xhi_ = std::min(mz_, xb_ + pz_);
  rlo_ = xa_;
  rhi_ = xb_ + 2 * pz_;
  if (world_ == 1) {
    xlo_ = 0;
    xhi_ = mz_;
  }
  // c0: >= 2p_x and a multiple of 32 floats (one 128-byte line), so x-shaped output tiles
  // cover whole lines and share none with their neighbours (a line written partly by two
  // CTAs at different times costs DRAM read-modify-writes: measured ~2x write traffic on
  // small PSFs at 16-byte alignment)
  X_ = Vol::make(xhi_ - xlo_, my_, mx_, 2 * py_, static_cast<int>(cdiv(2 * px_, 32) * 32));
  Y_ = Vol::make(rhi_ - rlo_, my_ + 2 * py_, mx_ + 2 * px_);
  if (!merged_) {
    xruns_.assign(1, {0, xa_n_});
    ny_user_planes_ = yb_ - ya_;
  }
  nreal_x_ = 1;
  for (size_t e : uext_x_) nreal_x_ *= static_cast<double>(e);

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    fail(NDC_ERR_NO_DEVICE, "ndconv_b200: no CUDA device (the device path has no CPU fallback)");
  }
  if (device < 0 || device >= ndev) fail(NDC_ERR_ARGUMENT, "ndconv_b200: bad device ordinal");
  check_cuda(cudaSetDevice(device_), "cudaSetDevice");
  cudaDeviceProp prop;
  check_cuda(cudaGetDeviceProperties(&prop, device_), "cudaGetDeviceProperties");
  if (prop.major != 10)
    fail(NDC_ERR_NO_DEVICE, std::string("ndconv_b200: built for sm_100a, device is ") + prop.name);
  check_cuda(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "cudaStreamCreate");
  check_cuda(cudaStreamCreateWithFlags(&edge_stream_, cudaStreamNonBlocking), "cudaStreamCreate");
  check_cuda(cudaEventCreateWithFlags(&fork_ev_, cudaEventDisableTiming), "cudaEventCreate");
  check_cuda(cudaEventCreateWithFlags(&join_ev_, cudaEventDisableTiming), "cudaEventCreate");
  if (world_ > 1) {
    check_cuda(cudaStreamCreateWithFlags(&comm_stream_, cudaStreamNonBlocking), "cudaStreamCreate");
    check_cuda(cudaEventCreateWithFlags(&pass_ev_, cudaEventDisableTiming), "cudaEventCreate");
    if (const char* e = std::getenv("NDC_HALO_OVERLAP")) halo_overlap_ = std::atoi(e) != 0;
  }
  alloc_all();
}

Plan::~Plan() {
  cudaSetDevice(device_);
  if (stream_) cudaStreamSynchronize(stream_);
  if (comm_stream_) cudaStreamSynchronize(comm_stream_);  // halo sends read plan buffers
  if (edge_stream_) cudaStreamSynchronize(edge_stream_);
  for (auto& e : ev_pool_) {
    cudaEventDestroy(e.first);
    cudaEventDestroy(e.second);
  }
  if (guard_mode()) {
    try {
      check_guards();
    } catch (...) {
    }
  }
  for (void* p : {static_cast<void*>(x_), static_cast<void*>(trial_), static_cast<void*>(g_),
                  static_cast<void*>(trial2_), static_cast<void*>(g2_),
                  static_cast<void*>(yobs_), static_cast<void*>(r_), static_cast<void*>(rt_),
                  static_cast<void*>(scratch_), static_cast<void*>(partials_),
                  static_cast<void*>(dsc_), static_cast<void*>(dscale_),
                  static_cast<void*>(dactive_), static_cast<void*>(dstep_), static_cast<void*>(gather_),
                  staging_})
    dfree(p);
  if (stream_) cudaStreamSynchronize(stream_);
  if (comm_stream_) cudaStreamSynchronize(comm_stream_);
  for (auto& e : halo_ev_)
    if (e.second) cudaEventDestroy(e.second);
  if (pass_ev_) cudaEventDestroy(pass_ev_);
  if (fork_ev_) cudaEventDestroy(fork_ev_);
  if (join_ev_) cudaEventDestroy(join_ev_);
  if (edge_stream_) cudaStreamDestroy(edge_stream_);
  if (comm_stream_) cudaStreamDestroy(comm_stream_);
  if (hsc_) small_pinned_put(small_bytes_, hsc_);
  if (up_ev_) cudaEventDestroy(up_ev_);
  if (d2h_ev_) cudaEventDestroy(d2h_ev_);
  release_pinned();
  if (stream_) cudaStreamDestroy(stream_);
}

// Device memory comes from the device's stream-ordered pool with the release threshold
// raised, so destroying and re-creating plans (every one-shot C-ABI call) reuses HBM
// instead of paying cudaMalloc / cudaFree each time.
unsigned long long guard_violations() { return g_guard_violations.load(); }

size_t Plan::check_guards() {
  if (allocs_.empty()) return 0;
  drain_halos();
  check_cuda(cudaStreamSynchronize(stream_), "cudaStreamSynchronize");
  if (edge_stream_) check_cuda(cudaStreamSynchronize(edge_stream_), "cudaStreamSynchronize");
  std::vector<unsigned char> h(kGuard);
  size_t bad = 0;
  for (const auto& a : allocs_) {
    for (int side = 0; side < 2; ++side) {
      const char* src = static_cast<const char*>(a.second.first) + (side ? kGuard + a.second.second : 0);
      check_cuda(cudaMemcpy(h.data(), src, kGuard, cudaMemcpyDeviceToHost), "D2H guard");
      for (unsigned char c : h) bad += c != kGuardByte;
    }
  }
  g_guard_violations += bad;
  return bad;
}

// Test hook for the checker itself: overwrite 16 bytes just past the observation buffer.
void Plan::debug_corrupt_guard() {
  auto it = allocs_.find(yobs_);
  if (!guard_mode() || it == allocs_.end()) fail(NDC_ERR_ARGUMENT, "guard bands are off (NDC_GUARD_BANDS=1)");
  check_cuda(cudaMemsetAsync(static_cast<char*>(it->first) + it->second.second, 0, 16, stream_), "cudaMemset");
}

void Plan::dfree(void* p) {
  if (p == nullptr) return;
  auto it = allocs_.find(p);
  if (it == allocs_.end()) {
    cudaFreeAsync(p, stream_);
    return;
  }
  cudaFreeAsync(it->second.first, stream_);
  allocs_.erase(it);
}

void* Plan::dmalloc(size_t bytes) {
  // once per device; plans of in-process slab ranks are created from concurrent threads
  static std::once_flag pool_set[64];
  if (device_ < 64)
    std::call_once(pool_set[device_], [this] {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, device_) == cudaSuccess) {
        uint64_t thr = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
      cudaGetLastError();
    });
  void* p = nullptr;
  if (guard_mode()) {
    check_cuda(cudaMallocAsync(&p, bytes + 2 * kGuard, stream_), "cudaMallocAsync");
    check_cuda(cudaMemsetAsync(p, kGuardByte, kGuard, stream_), "cudaMemset guard");
    check_cuda(cudaMemsetAsync(static_cast<char*>(p) + kGuard + bytes, kGuardByte, kGuard, stream_),
               "cudaMemset guard");
    void* user = static_cast<char*>(p) + kGuard;
    allocs_[user] = {p, bytes};
    return user;
  }
  check_cuda(cudaMallocAsync(&p, bytes, stream_), "cudaMallocAsync");
  return p;
}

float* Plan::dev_alloc_f(long long n) {
  void* p = dmalloc(static_cast<size_t>(n) * 4);
  check_cuda(cudaMemsetAsync(p, 0, static_cast<size_t>(n) * 4, stream_), "cudaMemset");
  return static_cast<float*>(p);
}

namespace {
// Persistent host worker pool for the host side of transfers: pageable <-> pinned
// memcpy (a single thread moves ~10 GB/s; the PCIe DMA it feeds is several times
// faster) and parallel pread / pwrite of tensor files.
class HostPool {
 public:
  static HostPool& get() {
    static HostPool pool;
    return pool;
  }
  unsigned width() const { return static_cast<unsigned>(workers_.size()) + 1; }
  // Runs fn(0) .. fn(parts-1) concurrently (the caller takes part 0); fn must not throw.
  void run(unsigned parts, const std::function<void(unsigned)>& fn) {
    if (parts <= 1) {
      fn(0);
      return;
    }
    std::unique_lock<std::mutex> call(call_mu_);  // one parallel job at a time
    {
      std::lock_guard<std::mutex> lk(mu_);
      fn_ = &fn;
      for (unsigned i = 1; i < parts; ++i) jobs_.push_back(i);
      pending_ += parts - 1;
    }
    cv_.notify_all();
    fn(0);
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return pending_ == 0; });
    fn_ = nullptr;
  }

 private:
  HostPool() {
    const unsigned hw = std::max(2u, std::thread::hardware_concurrency());
    for (unsigned i = 0; i + 1 < std::min(hw, 16u); ++i) workers_.emplace_back([this] { loop(); });
  }
  ~HostPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  void loop() {
    for (;;) {
      unsigned part;
      const std::function<void(unsigned)>* fn;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || !jobs_.empty(); });
        if (stop_) return;
        part = jobs_.back();
        jobs_.pop_back();
        fn = fn_;
      }
      (*fn)(part);
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_cv_.notify_all();
    }
  }
  std::vector<std::thread> workers_;
  std::vector<unsigned> jobs_;
  const std::function<void(unsigned)>* fn_ = nullptr;
  std::mutex mu_, call_mu_;
  std::condition_variable cv_, done_cv_;
  size_t pending_ = 0;
  bool stop_ = false;
};

// Splits [0, n) into `parts` near-equal ranges.
inline std::pair<size_t, size_t> part_range(size_t n, unsigned parts, unsigned i) {
  const size_t per = (n + parts - 1) / parts;
  return {std::min(n, i * per), std::min(n, (i + 1) * per)};
}

void par_copy(void* dst, const void* src, size_t n) {
  const unsigned parts = static_cast<unsigned>(std::min<size_t>(HostPool::get().width(), n >> 20));
  HostPool::get().run(std::max(1u, parts), [&](unsigned i) {
    const auto r = part_range(n, std::max(1u, parts), i);
    std::memcpy(static_cast<char*>(dst) + r.first, static_cast<const char*>(src) + r.first, r.second - r.first);
  });
}


constexpr size_t kPinChunk = size_t(16) << 20;

// Pinned staging rings are cached per process (cudaMallocHost / cudaFreeHost are slow
// and would otherwise be paid by every one-shot call).
struct PinnedRing {
  void* buf[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
};
std::mutex g_ring_mu;
std::vector<PinnedRing> g_rings;

// Small pinned blocks (per-plan scalar mirrors), cached per process by size.
std::mutex g_small_mu;
std::vector<std::pair<size_t, void*>> g_small;
void* small_pinned_get(size_t bytes) {
  {
    std::lock_guard<std::mutex> lk(g_small_mu);
    for (size_t i = 0; i < g_small.size(); ++i)
      if (g_small[i].first == bytes) {
        void* p = g_small[i].second;
        g_small.erase(g_small.begin() + static_cast<long>(i));
        return p;
      }
  }
  void* p = nullptr;
  check_cuda(cudaMallocHost(&p, bytes), "cudaMallocHost scalars");
  return p;
}
void small_pinned_put(size_t bytes, void* p) {
  std::lock_guard<std::mutex> lk(g_small_mu);
  g_small.emplace_back(bytes, p);
}
}  // namespace

void Plan::ensure_pinned() {
  if (hpin_[0]) return;
  PinnedRing r;
  {
    std::lock_guard<std::mutex> lk(g_ring_mu);
    if (!g_rings.empty()) {
      r = g_rings.back();
      g_rings.pop_back();
    }
  }
  if (!r.buf[0]) {
    for (int i = 0; i < 2; ++i) {
      check_cuda(cudaMallocHost(&r.buf[i], kPinChunk), "cudaMallocHost staging");
      check_cuda(cudaEventCreateWithFlags(&r.ev[i], cudaEventDisableTiming), "cudaEventCreate");
    }
  }
  for (int i = 0; i < 2; ++i) {
    hpin_[i] = r.buf[i];
    pin_ev_[i] = r.ev[i];
  }
}

void Plan::release_pinned() {
  if (!hpin_[0]) return;
  PinnedRing r;
  for (int i = 0; i < 2; ++i) {
    r.buf[i] = hpin_[i];
    r.ev[i] = pin_ev_[i];
    hpin_[i] = nullptr;
    pin_ev_[i] = nullptr;
  }
  std::lock_guard<std::mutex> lk(g_ring_mu);
  g_rings.push_back(r);
}

// Host (pageable) -> device through a double-buffered pinned ring: host threads fill
// one 16 MB slot while the DMA of the other runs.
void Plan::h2d_staged(void* dev, const void* host, size_t bytes) {
  if (bytes < (size_t(4) << 20)) {
    check_cuda(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, stream_), "H2D");
    return;
  }
  ensure_pinned();
  size_t i = 0;
  for (size_t off = 0; off < bytes; off += kPinChunk, ++i) {
    const int s = static_cast<int>(i & 1);
    const size_t n = std::min(kPinChunk, bytes - off);
    // the slot may still feed a DMA of this call or of an earlier one (any call starts
    // at slot 0): wait for its last use before the host overwrites it
    check_cuda(cudaEventSynchronize(pin_ev_[s]), "cudaEventSynchronize");
    par_copy(hpin_[s], static_cast<const char*>(host) + off, n);
    check_cuda(cudaMemcpyAsync(static_cast<char*>(dev) + off, hpin_[s], n, cudaMemcpyHostToDevice,
                               stream_),
               "H2D");
    check_cuda(cudaEventRecord(pin_ev_[s], stream_), "cudaEventRecord");
  }
}

// Device -> host (pageable): the DMA of chunk i+1 overlaps the host copy-out of chunk i.
void Plan::d2h_staged(void* host, const void* dev, size_t bytes) {
  if (bytes < (size_t(4) << 20)) {
    check_cuda(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, stream_), "D2H");
    sync();
    return;
  }
  ensure_pinned();
  const size_t nch = (bytes + kPinChunk - 1) / kPinChunk;
  auto issue = [&](size_t i) {
    const int s = static_cast<int>(i & 1);
    const size_t off = i * kPinChunk, n = std::min(kPinChunk, bytes - off);
    check_cuda(cudaMemcpyAsync(hpin_[s], static_cast<const char*>(dev) + off, n,
                               cudaMemcpyDeviceToHost, stream_),
               "D2H");
    check_cuda(cudaEventRecord(pin_ev_[s], stream_), "cudaEventRecord");
  };
  if (nch == 0) return;
  issue(0);
  for (size_t i = 0; i < nch; ++i) {
    if (i + 1 < nch) issue(i + 1);
    const int s = static_cast<int>(i & 1);
    check_cuda(cudaEventSynchronize(pin_ev_[s]), "cudaEventSynchronize");
    const size_t off = i * kPinChunk, n = std::min(kPinChunk, bytes - off);
    par_copy(static_cast<char*>(host) + off, hpin_[s], n);
  }
}

long long Plan::partials_per_image(Dir d) const {
  const Vol& vo = (d == kFwd) ? Y_ : X_;
  const long long nz = (d == kFwd) ? (yb_ - ya_) : (xb_ - xa_);
  return nz * cdiv(vo.ex, kTileX) * cdiv(vo.ey, kTileY * ry_) * (kThreads / 32);  // per warp
}

void Plan::alloc_all() {
  const long long nx = X_.image * static_cast<long long>(B_);
  const long long ny = Y_.image * static_cast<long long>(B_);
  x_ = dev_alloc_f(nx);
  trial_ = dev_alloc_f(nx);
  g_ = dev_alloc_f(nx);
  yobs_ = dev_alloc_f(ny);
  r_ = dev_alloc_f(ny);
  rt_ = dev_alloc_f(ny);
  // partial sums of multi-launch (chunked) PSFs, see correlate()
  const bool chunked = chunks_fwd_.size() > 1 || chunks_adj_.size() > 1;
  if (chunked) scratch_ = dev_alloc_f(std::max(nx, ny));
  partials_cap_ = static_cast<long long>(B_) *
                  std::max({partials_per_image(kFwd), partials_per_image(kAdj),
                            static_cast<long long>(kElemBlocks)});
  partials_ = static_cast<double2*>(dmalloc(partials_cap_ * sizeof(double2)));
  const size_t nsc = kNumSlots * B_ + kMaxPowerIters + 16;
  dsc_ = static_cast<double*>(dmalloc(nsc * sizeof(double)));
  check_cuda(cudaMemsetAsync(dsc_, 0, nsc * sizeof(double), stream_), "cudaMemset");
  // pinned scalar mirrors: [nsc doubles of D2H results][B steps][B active flags]
  small_bytes_ = ((nsc + B_) * sizeof(double) + B_ * sizeof(int) + 4095) / 4096 * 4096;
  hsc_ = static_cast<double*>(small_pinned_get(small_bytes_));
  hstep_ = hsc_ + nsc;
  hact_ = reinterpret_cast<int*>(hstep_ + B_);
  check_cuda(cudaEventCreateWithFlags(&up_ev_, cudaEventDisableTiming), "cudaEventCreate");
  check_cuda(cudaEventCreateWithFlags(&d2h_ev_, cudaEventDisableTiming), "cudaEventCreate");
  dscale_ = static_cast<float*>(dmalloc(B_ * sizeof(float)));
  dactive_ = static_cast<int*>(dmalloc(B_ * sizeof(int)));
  dstep_ = static_cast<double*>(dmalloc(B_ * sizeof(double)));
  if (comm_) gather_ = static_cast<double*>(dmalloc(2 * world_ * sizeof(double)));
  std::vector<float> ones(B_, 1.0f);
  check_cuda(cudaMemcpyAsync(dscale_, ones.data(), B_ * 4, cudaMemcpyHostToDevice, stream_), "H2D");
  std::vector<int> act(B_, 1);
  check_cuda(cudaMemcpyAsync(dactive_, act.data(), B_ * 4, cudaMemcpyHostToDevice, stream_), "H2D");
  act_cache_ = act;
  staging_bytes_ = static_cast<size_t>(std::max(X_.ez * static_cast<long long>(X_.ey) * X_.ex,
                                                Y_.ez * static_cast<long long>(Y_.ey) * Y_.ex)) * 8;
  staging_ = dmalloc(staging_bytes_);
  sync();
}

void Plan::sync() {
  drain_halos();  // the plan stream then covers the comm stream too
  check_cuda(cudaStreamSynchronize(stream_), "cudaStreamSynchronize");
}

const CUtensorMap& Plan::map_for(const float* base, Dir d, int sh, int kx, int ky) {
  auto key = std::make_pair(base, static_cast<int>(d) + 2 * (kx + 64 * ky));
  auto it = maps_.find(key);
  if (it != maps_.end()) return it->second;
  const Vol& v = (d == kFwd) ? X_ : Y_;
  CUtensorMap m;
  // x-shaped inputs are described including their zero margin (ndc_plan.h Vol)
  const CUresult rc = encode_tensor_map(&m, base, v.c0 + v.ex, v.r0 + v.ey,
                                        static_cast<long long>(v.ez) * B_, v.pitch, v.plane,
                                        shared_pitch_for(kx, sh), kTileY * ry_ + ky - 1);
  if (rc != CUDA_SUCCESS)
    fail(NDC_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(rc)) + ")");
  return maps_.emplace(key, m).first->second;
}

void Plan::correlate(Dir d, const float* in, float* out, int mode, float* aux_out,
                     const float* aux_in, const float* scale, const double* step, const int* active,
                     bool partials) {
  const bool fwd = d == kFwd;
  const Vol& vin = fwd ? X_ : Y_;
  const Vol& vout = fwd ? Y_ : X_;
  const std::vector<float>& taps = fwd ? taps_fwd_ : taps_adj_;
  CorrGeom g{};
  g.in_ez = vin.ez;
  g.out_ey = vout.ey;
  g.out_ex = vout.ex;
  int nz_out;
  int sh = 0;
  if (fwd) {
    nz_out = yb_ - ya_;
    g.out_z0 = ya_ - rlo_;
    g.off_z = ya_ - 2 * pz_ - xlo_;
    g.off_y = X_.r0 - 2 * py_;
    sh = (X_.c0 - 2 * px_) & 3;  // 0 or 2 (2p is even, c0 a multiple of 4)
    g.off_x = X_.c0 - 2 * px_ - sh;
  } else {
    nz_out = xb_ - xa_;
    g.out_z0 = xa_ - xlo_;
    g.off_z = xa_ - rlo_;
    g.off_y = 0;
    g.off_x = 0;
  }
  // TMA tile starts must be non-negative (x-shaped inputs carry a zero margin)
  if (g.off_x < 0 || g.off_y < 0 || (g.off_x & 3))
    fail(NDC_ERR_CUDA, "internal: negative or unaligned TMA tile origin");
  g.tiles_x = static_cast<int>(cdiv(vout.ex, kTileX));
  g.tiles_y = static_cast<int>(cdiv(vout.ey, kTileY * ry_));
  // partial edge tiles run as a second launch with the edge kernel (ndc_correlate.cuh);
  // HBM-bound small PSFs keep one launch (the edge kernel's gain is compute-side)
  g.full_tx = KX_ <= kSmallMaxKX ? g.tiles_x : vout.ex / kTileX;
  g.full_ty = KX_ <= kSmallMaxKX ? g.tiles_y : vout.ey / (kTileY * ry_);
  g.out_pitch = vout.pitch;
  g.out_plane = vout.plane;
  g.out_image = vout.image;
  g.mode = mode;
  const int off_x0 = g.off_x, off_y0 = g.off_y;
  const int kxp_full = tap_pitch(KX_);
  const std::vector<TapChunk>& chunks = fwd ? chunks_fwd_ : chunks_adj_;
  static thread_local TapBlock tb;
  // One launch per tap chunk and plane segment [z_base, z_base + nz) of the computed
  // planes.  A segment that does not start at plane 0 shifts the output / input plane
  // offsets and the partials pointer (single-image slab plans only), so the kernel's
  // plane index stays blockIdx.y.
  // Partial edge tiles run on the side stream (fork / join around the whole pass), so
  // their CTAs fill the SMs the full-tile launch frees in its last wave; each stream keeps
  // its tap chunks in order, and the two touch disjoint output tiles.
  const bool side = g.tiles_x * g.tiles_y > g.full_tx * g.full_ty && g.full_tx * g.full_ty > 0;
  const int out_z0_base = g.out_z0, off_z_base = g.off_z;
  const long long part_per_plane = static_cast<long long>(g.tiles_x) * g.tiles_y * (kThreads / 32);
  struct Seg {
    int z_base, nz;
  };
  auto run_chunks = [&](const std::vector<Seg>& segs) {
    size_t ev = 0;
    if (timing_) {
      if (ev_used_ == ev_pool_.size()) {
        cudaEvent_t e0, e1;
        check_cuda(cudaEventCreate(&e0), "cudaEventCreate");
        check_cuda(cudaEventCreate(&e1), "cudaEventCreate");
        ev_pool_.emplace_back(e0, e1);
      }
      ev = ev_used_++;
      check_cuda(cudaEventRecord(ev_pool_[ev].first, stream_), "cudaEventRecord");
    }
    if (side) {
      check_cuda(cudaEventRecord(fork_ev_, stream_), "cudaEventRecord");
      check_cuda(cudaStreamWaitEvent(edge_stream_, fork_ev_, 0), "cudaStreamWaitEvent");
    }
    for (const Seg& sg : segs) {
      if (sg.nz <= 0) continue;
      if (sg.z_base != 0 && B_ != 1) fail(NDC_ERR_CUDA, "internal: plane segments need a single-image plan");
      g.out_z0 = out_z0_base + sg.z_base;
      g.off_z = off_z_base + sg.z_base;
      for (size_t c = 0; c < chunks.size(); ++c) {
        const TapChunk& ch = chunks[c];
        g.KY = ch.cy;
        g.rows = kTileY * ry_ + ch.cy - 1;
        g.pitch_s = shared_pitch_for(ch.w, sh);
        g.off_x = off_x0 + ch.kx0;  // multiples of 32: the TMA origin stays 16-byte aligned
        g.off_y = off_y0 + ch.ky0;
        g.kz0 = ch.kz0;
        g.kz1 = ch.kz1;
        g.stages = std::min(stages_, g.kz1 - g.kz0);
        g.aux_prefetch = (KZ_ == 1 && (KX_ <= kStagedMaxKX || KX_ <= kPrefetchMaxKX)) ? 1 : 0;
        g.accum = c > 0;
        g.final_chunk = (c + 1 == chunks.size());
        // x-shaped operands are addressed from their interior origin
        const long long xo = fwd ? 0 : X_.origin;
        auto at = [xo](const float* p) { return p ? const_cast<float*>(p) + xo : nullptr; };
        CorrArgs a{};
        a.out = at(g.final_chunk ? out : scratch_);
        a.accum_in = at(scratch_);
        a.aux_out = at(aux_out);
        a.aux_in = fwd ? aux_in : at(aux_in);
        a.scale = scale;
        a.step = step;
        a.active = active;
        a.partials = (g.final_chunk && partials) ? partials_ + sg.z_base * part_per_plane : nullptr;
        // gather the chunk's taps [kz][ky][kx] with row pitch tap_pitch(w), zero padded
        const int wp = tap_pitch(ch.w);
        if (ch.kx0 == 0 && ch.w == KX_ && ch.cy == KY_) {
          std::memcpy(tb.t, taps.data() + static_cast<size_t>(ch.kz0) * KY_ * kxp_full,
                      static_cast<size_t>(ch.kz1 - ch.kz0) * KY_ * kxp_full * sizeof(float));
        } else {
          for (int kz = ch.kz0; kz < ch.kz1; ++kz)
            for (int ky = 0; ky < ch.cy; ++ky) {
              float* dst = tb.t + (static_cast<size_t>(kz - ch.kz0) * ch.cy + ky) * wp;
              const float* src = taps.data() + (static_cast<size_t>(kz) * KY_ + ch.ky0 + ky) * kxp_full + ch.kx0;
              for (int kx = 0; kx < wp; ++kx) dst[kx] = kx < ch.cw ? src[kx] : 0.0f;
            }
        }
        const CUtensorMap& map = map_for(in, d, sh, ch.w, ch.cy);
        check_cuda(launch_correlate(ch.w, sh, ry_, map, g, a, tb, static_cast<int>(B_), sg.nz, stream_,
                                    side ? edge_stream_ : stream_),
                   "correlate launch");
        // kernels launched: full tiles and / or the edge tiles
        const int nk = (g.full_tx * g.full_ty > 0 ? 1 : 0) + (g.tiles_x * g.tiles_y > g.full_tx * g.full_ty ? 1 : 0);
        st_[fwd ? 0 : 1].launches += nk;
        st_[2].launches += nk;
      }
    }
    if (side) {
      check_cuda(cudaEventRecord(join_ev_, edge_stream_), "cudaEventRecord");
      check_cuda(cudaStreamWaitEvent(stream_, join_ev_, 0), "cudaStreamWaitEvent");
    }
    if (timing_) {
      check_cuda(cudaEventRecord(ev_pool_[ev].second, stream_), "cudaEventRecord");
      ev_pending_.emplace_back(fwd ? 0 : 1, ev);
    }
  };
  // Outputs still being sent to a neighbour, or halo planes still arriving, must not be
  // overwritten: wait for their exchange first (no-op unless an exchange is pending).
  wait_halo(out);
  wait_halo(aux_out);
  // z-slab ranks: the first `lo` / last `hi` computed planes are exactly the planes that
  // read the input's halo and the planes the neighbours need next, so the
  // other planes run first, before waiting for the input's halo exchange (which overlaps
  // them), then the boundary planes.
  const int lo = (world_ > 1 && rank_ > 0) ? pz_ : 0;
  const int hi = (world_ > 1 && rank_ + 1 < world_) ? pz_ : 0;
  const int n_int = nz_out - lo - hi;
  if (merged_ && !fwd) {
    // x-shaped outputs of a merged (ndim > 3) plan: only x's real planes; the partial
    // slots of the skipped planes are zeroed so the per-pass reductions ignore them
    if (partials)
      check_cuda(cudaMemsetAsync(partials_, 0, partials_per_image(kAdj) * sizeof(double2), stream_),
                 "cudaMemset partials");
    std::vector<Seg> segs;
    for (const auto& r : xruns_) segs.push_back({r.first, r.second});
    wait_halo(in);
    run_chunks(segs);
  } else if (halo_overlap_ && (lo + hi) > 0 && n_int > 0) {
    run_chunks({{lo, n_int}});
    wait_halo(in);
    run_chunks({{0, lo}, {nz_out - hi, hi}});
  } else {
    wait_halo(in);
    run_chunks({{0, nz_out}});
  }
}

void Plan::drain_events() {
  if (ev_pending_.empty()) return;
  sync();
  for (auto& pe : ev_pending_) {
    float ms = 0.f;
    check_cuda(cudaEventElapsedTime(&ms, ev_pool_[pe.second].first, ev_pool_[pe.second].second),
               "cudaEventElapsedTime");
    st_[pe.first].ms += ms;
  }
  ev_pending_.clear();
  ev_used_ = 0;
}

void Plan::reset_stats() {
  drain_events();
  for (auto& s : st_) s = KernelStats{};
}

KernelStats Plan::stats(int kind) {
  drain_events();
  if (kind < 0 || kind > 2) fail(NDC_ERR_ARGUMENT, "stats kind");
  return st_[kind];
}

void Plan::finalize(long long per_image, int op, double* out0, double* out1, float* scale_out,
                    const int* active) {
  if (!comm_) {
    check_cuda(launch_finalize(partials_, per_image, static_cast<int>(B_), op, out0, out1, scale_out,
                               active, stream_),
               "finalize launch");
    st_[2].launches++;
    return;
  }
  // z-slab ranks: raw local reduction -> all-gather (rank order) -> identical combine
  // (a one-rank transport runs the same sequence: its all-gather is a real NCCL call).
  const int raw = (op == kFinMaxSum) ? kFinMaxSum : kFinSumSum;
  double* gin = dsc_ + kNumSlots * B_ + kMaxPowerIters;  // 2 doubles
  double* gout = gather_;                                 // 2 * world doubles
  check_cuda(launch_finalize(partials_, per_image, 1, raw, gin, gin + 1, nullptr, active, stream_),
             "finalize launch");
  comm_->allgather(gin, gout, 2, stream_);
  check_cuda(launch_combine(gout, world_, op, out0, out1, scale_out, stream_), "combine launch");
  st_[2].launches += 2;
}

// Halo planes: the forward pass needs p_z x-planes from each neighbour,
// the adjoint p_z y-planes; slabs are at least p_z thick so one neighbour suffices.
//
// halo_x / halo_y enqueue the exchange of `buf`'s boundary planes on the comm stream once
// everything enqueued so far on the plan stream is done, and record a per-buffer event.
// The plan stream does not wait for it: correlate() waits before the launch that reads
// the halo (after the planes that do not need it), and before any launch that writes
// `buf`; every other user of a sharded buffer drains the pending exchanges first
// (drain_halos).  With NDC_HALO_OVERLAP=0 the plan stream waits right away (the exchange
// is serialised with the passes, as a plain send/recv would be).
void Plan::halo_x(float* buf) {
  if (world_ == 1 || pz_ == 0) return;
  const size_t n = static_cast<size_t>(pz_) * X_.plane;
  auto at = [&](int global_plane) { return buf + static_cast<long long>(global_plane - xlo_) * X_.plane; };
  const bool lo = rank_ > 0, hi = rank_ + 1 < world_;
  halo_enqueue(buf, lo ? at(xa_) : nullptr, lo ? at(xa_ - pz_) : nullptr, hi ? at(xb_ - pz_) : nullptr,
               hi ? at(xb_) : nullptr, n);
}

void Plan::halo_y(float* buf) {
  if (world_ == 1 || pz_ == 0) return;
  const size_t n = static_cast<size_t>(pz_) * Y_.plane;
  auto at = [&](int global_plane) { return buf + static_cast<long long>(global_plane - rlo_) * Y_.plane; };
  const bool lo = rank_ > 0, hi = rank_ + 1 < world_;
  halo_enqueue(buf, lo ? at(xa_ + pz_) : nullptr, lo ? at(xa_) : nullptr, hi ? at(xb_) : nullptr,
               hi ? at(xb_ + pz_) : nullptr, n);
}

void Plan::halo_enqueue(const float* buf, const float* send_lo, float* recv_lo, const float* send_hi,
                        float* recv_hi, size_t n) {
  wait_halo(buf);  // an earlier exchange of the same buffer (its planes are rewritten now)
  check_cuda(cudaEventRecord(pass_ev_, stream_), "cudaEventRecord");
  check_cuda(cudaStreamWaitEvent(comm_stream_, pass_ev_, 0), "cudaStreamWaitEvent");
  comm_->exchange(send_lo, recv_lo, send_hi, recv_hi, n, comm_stream_);
  cudaEvent_t& ev = halo_ev_[buf];
  if (ev == nullptr) check_cuda(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "cudaEventCreate");
  check_cuda(cudaEventRecord(ev, comm_stream_), "cudaEventRecord");
  halo_pending_.insert(buf);
  if (!halo_overlap_) wait_halo(buf);
}

void Plan::wait_halo(const float* buf) {
  if (buf == nullptr || halo_pending_.empty()) return;
  auto it = halo_pending_.find(buf);
  if (it == halo_pending_.end()) return;
  check_cuda(cudaStreamWaitEvent(stream_, halo_ev_[buf], 0), "cudaStreamWaitEvent");
  halo_pending_.erase(it);
}

void Plan::drain_halos() {
  while (!halo_pending_.empty()) wait_halo(*halo_pending_.begin());
}

// Per-image flags / steps go to the device only when they change (they rarely do), from
// pinned mirrors, without a stream sync; up_ev_ guards the mirror against reuse while
// an earlier upload is still in flight.
void Plan::upload_active(const std::vector<int>& act) {
  if (act == act_cache_) return;
  check_cuda(cudaEventSynchronize(up_ev_), "cudaEventSynchronize");
  std::memcpy(hact_, act.data(), act.size() * sizeof(int));
  check_cuda(cudaMemcpyAsync(dactive_, hact_, act.size() * sizeof(int), cudaMemcpyHostToDevice, stream_),
             "H2D active");
  check_cuda(cudaEventRecord(up_ev_, stream_), "cudaEventRecord");
  act_cache_ = act;
}

void Plan::upload_steps(const std::vector<double>& steps) {
  if (steps == step_cache_) return;
  check_cuda(cudaEventSynchronize(up_ev_), "cudaEventSynchronize");
  std::memcpy(hstep_, steps.data(), steps.size() * sizeof(double));
  check_cuda(cudaMemcpyAsync(dstep_, hstep_, steps.size() * sizeof(double), cudaMemcpyHostToDevice, stream_),
             "H2D steps");
  check_cuda(cudaEventRecord(up_ev_, stream_), "cudaEventRecord");
  step_cache_ = steps;
}

// ---- host <-> device packing (dense row-major host, pitched device) -----------------
namespace {
// dst[i] = float(src[i]) / double(src[i]) over the host pool (round to nearest: the same
// value the device conversion would give).
template <class D, class S>
void par_convert(D* dst, const S* src, size_t n) {
  const unsigned parts = static_cast<unsigned>(std::max<size_t>(1, std::min<size_t>(HostPool::get().width(), n >> 18)));
  HostPool::get().run(parts, [&](unsigned i) {
    const auto r = part_range(n, parts, i);
    for (size_t k = r.first; k < r.second; ++k) dst[k] = static_cast<D>(src[k]);
  });
}
}  // namespace

// f64 host -> f32 device: host threads convert into the pinned ring (half the PCIe
// bytes of shipping f64 and converting on the device; identical values).
void Plan::h2d_f64_as_f32(float* dev, const double* host, size_t n) {
  ensure_pinned();
  const size_t chunk = kPinChunk / 4;
  size_t i = 0;
  for (size_t off = 0; off < n; off += chunk, ++i) {
    const int s = static_cast<int>(i & 1);
    const size_t m = std::min(chunk, n - off);
    // the slot may still feed a DMA of this call or of an earlier one (any call starts
    // at slot 0): wait for its last use before the host overwrites it
    check_cuda(cudaEventSynchronize(pin_ev_[s]), "cudaEventSynchronize");
    par_convert(static_cast<float*>(hpin_[s]), host + off, m);
    check_cuda(cudaMemcpyAsync(dev + off, hpin_[s], m * 4, cudaMemcpyHostToDevice, stream_), "H2D");
    check_cuda(cudaEventRecord(pin_ev_[s], stream_), "cudaEventRecord");
  }
}

void Plan::pack_dense_f64(const double* host, float* dev, const Vol& v, int z_off, int nz) {
  drain_halos();
  const size_t per = static_cast<size_t>(nz) * v.ey * v.ex;
  // f64 -> f32 on the host threads, then f32 over PCIe (measured 13.8 vs 15.7 ms for the
  // config-2 batch against the f64 DMA + device conversion)
  const bool big = per * 8 >= (size_t(4) << 20);
  for (size_t b = 0; b < B_; ++b) {
    if (big) {
      h2d_f64_as_f32(static_cast<float*>(staging_), host + b * per, per);
      check_cuda(launch_pack_f32(static_cast<const float*>(staging_),
                                 dev + b * v.image + v.origin + static_cast<long long>(z_off) * v.plane, 1,
                                 v.geo(nz), stream_),
                 "pack");
    } else {
      h2d_staged(staging_, host + b * per, per * 8);
      check_cuda(launch_pack_f64(static_cast<const double*>(staging_),
                                 dev + b * v.image + v.origin + static_cast<long long>(z_off) * v.plane, 1,
                                 v.geo(nz), stream_),
                 "pack");
    }
    st_[2].launches++;
  }
  sync();
}

void Plan::pack_dense_f32(const float* host, float* dev, const Vol& v, int z_off, int nz) {
  drain_halos();
  const size_t per = static_cast<size_t>(nz) * v.ey * v.ex;
  for (size_t b = 0; b < B_; ++b) {
    h2d_staged(staging_, host + b * per, per * 4);
    check_cuda(launch_pack_f32(static_cast<const float*>(staging_),
                               dev + b * v.image + v.origin + static_cast<long long>(z_off) * v.plane, 1,
                               v.geo(nz), stream_),
               "pack");
    st_[2].launches++;
  }
  sync();
}

void Plan::unpack_dense_f64(const float* dev, double* host, const Vol& v, int z_off, int nz) {
  drain_halos();
  const size_t per = static_cast<size_t>(nz) * v.ey * v.ex;
  // Device-side f32 -> f64 conversion + f64 DMA + parallel memcpy out of the pinned ring:
  // measured faster than converting on the host (19 vs 31 ms for 16 x 2048^2 on the
  // 16-core box: the host conversion is bound by host memory bandwidth).
  for (size_t b = 0; b < B_; ++b) {
    check_cuda(launch_unpack_f64(dev + b * v.image + v.origin + static_cast<long long>(z_off) * v.plane,
                                 static_cast<double*>(staging_), 1, v.geo(nz), stream_),
               "unpack");
    st_[2].launches++;
    d2h_staged(host + b * per, staging_, per * 8);
  }
}

void Plan::unpack_dense_f32(const float* dev, float* host, const Vol& v, int z_off, int nz) {
  drain_halos();
  const size_t per = static_cast<size_t>(nz) * v.ey * v.ex;
  for (size_t b = 0; b < B_; ++b) {
    check_cuda(launch_unpack_f32(dev + b * v.image + v.origin + static_cast<long long>(z_off) * v.plane,
                                 static_cast<float*>(staging_), 1, v.geo(nz), stream_),
               "unpack");
    st_[2].launches++;
    d2h_staged(host + b * per, staging_, per * 4);
  }
}

void Plan::set_observation_f64(const double* y) {
  pack_dense_f64(y, yobs_, Y_, ya_ - rlo_, ny_user_planes_);
  halo_y(yobs_);
}
void Plan::set_observation_f32(const float* y) {
  pack_dense_f32(y, yobs_, Y_, ya_ - rlo_, ny_user_planes_);
  halo_y(yobs_);
}
void Plan::set_x_f64(const double* x) {
  for (size_t r = 0; r < xruns_.size(); ++r)
    pack_dense_f64(x + r * xrun_elems(), x_, X_, xa_ - xlo_ + xruns_[r].first, xruns_[r].second);
  halo_x(x_);
}
void Plan::set_x_f32(const float* x) {
  for (size_t r = 0; r < xruns_.size(); ++r)
    pack_dense_f32(x + r * xrun_elems(), x_, X_, xa_ - xlo_ + xruns_[r].first, xruns_[r].second);
  halo_x(x_);
}
void Plan::get_y_buffer_f32(float* y) { unpack_dense_f32(r_, y, Y_, ya_ - rlo_, ny_user_planes_); }
void Plan::get_x_buffer_f32(float* x) {
  for (size_t r = 0; r < xruns_.size(); ++r)
    unpack_dense_f32(x_, x + r * xrun_elems(), X_, xa_ - xlo_ + xruns_[r].first, xruns_[r].second);
}
void Plan::get_estimate_f64(double* x) {
  for (size_t r = 0; r < xruns_.size(); ++r)
    unpack_dense_f64(x_, x + r * xrun_elems(), X_, xa_ - xlo_ + xruns_[r].first, xruns_[r].second);
}
void Plan::get_estimate_f32(float* x) { get_x_buffer_f32(x); }
void Plan::get_observation_f64(double* y) { unpack_dense_f64(yobs_, y, Y_, ya_ - rlo_, ny_user_planes_); }
void Plan::get_y_buffer_f64(double* y) { unpack_dense_f64(r_, y, Y_, ya_ - rlo_, ny_user_planes_); }
void Plan::get_x_buffer_f64(double* x, int which) {
  for (size_t r = 0; r < xruns_.size(); ++r)
    unpack_dense_f64(which == 0 ? x_ : g_, x + r * xrun_elems(), X_, xa_ - xlo_ + xruns_[r].first,
                     xruns_[r].second);
}

// ---- operators ------------------------------------------------------------------------
void Plan::op_conv_full() {
  correlate(kFwd, x_, r_, kEpiStore, nullptr, nullptr, nullptr, nullptr, nullptr, false);
}

void Plan::op_adjoint_of_y() {
  correlate(kAdj, yobs_, x_, kEpiStore, nullptr, nullptr, nullptr, nullptr, nullptr, false);
}

double Plan::op_objective() {
  correlate(kFwd, x_, r_, kEpiResid, nullptr, yobs_, nullptr, nullptr, nullptr, true);
  finalize(partials_per_image(kFwd), kFinHalfSum, dsc_ + kF * B_, nullptr, nullptr, nullptr);
  check_cuda(cudaMemcpyAsync(hsc_, dsc_ + kF * B_, B_ * 8, cudaMemcpyDeviceToHost, stream_), "D2H");
  sync();
  return hsc_[0];
}

void Plan::op_normal_gradient() {
  op_objective();
  halo_y(r_);
  correlate(kAdj, r_, g_, kEpiStore, nullptr, nullptr, nullptr, nullptr, nullptr, false);
}

double Plan::op_kkt_residual() {
  op_objective();
  halo_y(r_);
  correlate(kAdj, r_, nullptr, kEpiKKT, nullptr, x_, nullptr, nullptr, nullptr, true);
  finalize(partials_per_image(kAdj), kFinMaxSum, dsc_ + kKKT * B_, dsc_ + kCHG * B_, nullptr,
           nullptr);
  check_cuda(cudaMemcpyAsync(hsc_, dsc_ + kKKT * B_, B_ * 8, cudaMemcpyDeviceToHost, stream_), "D2H");
  sync();
  return hsc_[0];
}

// solvers.hpp:127-143.  Run on image 0 only (the estimate depends on (h, shape) alone,
// so every image of a batch shares it); v_i = w_{i-1}/lambda_{i-1} is folded into the
// next forward pass as an output scale read on the device, so the 2*iters passes run
// without a host round trip.
double Plan::estimate_step(size_t power_iters) {
  if (estimate_pending_ == power_iters) return estimate_collect();
  estimate_launch(power_iters);
  return estimate_collect();
}

// The power iteration's passes and the read-back of every iterate's norm are only
// enqueued here; estimate_collect() waits.  The one-shot C-ABI calls launch it before
// they upload the observation (it needs only the PSF and the shape), so the host-side
// conversion of Y overlaps these device passes.
void Plan::estimate_launch(size_t power_iters) {
  drain_halos();
  if (power_iters == 0) fail(NDC_ERR_CONFIG, "estimate_step: power_iters must be positive");
  if (kernel_all_zero_) fail(NDC_ERR_NUMERIC, "estimate_step: degenerate all-zero kernel");
  const double n = nreal_x_;
  estimate_pending_ = 0;
  // Small problems run the power iteration in float64: when all-ones is an exact but
  // non-dominant eigenvector of A^T A (symmetric tiny shapes), the reference's f64
  // iteration stays in that eigenspace and float32 rounding would not.
  const char* sep_env = std::getenv("NDC_SEPARABLE_STEP");  // 0: off, 2: also small problems (tests)
  const bool sep_small = sep_env != nullptr && std::atoi(sep_env) == 2;
  if (world_ == 1 && !merged_ && n * static_cast<double>(h64_.size()) <= static_cast<double>(1 << 28) &&
      !(sep_small && estimate_step_separable(power_iters, &estimate_value_))) {
    estimate_value_ = estimate_step_f64(power_iters);
    estimate_pending_ = power_iters;
    estimate_f64_ = true;
    return;
  }
  // Separable PSFs (every BASELINE config but 5): exact factorisation, no device passes.
  if (estimate_step_separable(power_iters, &estimate_value_)) {
    estimate_pending_ = power_iters;
    estimate_f64_ = true;
    return;
  }
  const size_t saveB = B_;
  // image 0 only: launch with batch 1 (buffers are laid out image-major)
  B_ = 1;
  try {
    const float one = 1.0f;
    check_cuda(cudaMemcpyAsync(dscale_, &one, 4, cudaMemcpyHostToDevice, stream_), "H2D");
    fill_x_real(g_, 0, static_cast<float>(1.0 / std::sqrt(n)));
    double* lam = dsc_ + kNumSlots * saveB;
    for (size_t i = 0; i < power_iters; ++i) {
      halo_x(g_);
      correlate(kFwd, g_, rt_, kEpiStore, nullptr, nullptr, dscale_, nullptr, nullptr, false);
      halo_y(rt_);
      correlate(kAdj, rt_, g_, kEpiNorm, nullptr, nullptr, nullptr, nullptr, nullptr, true);
      finalize(partials_per_image(kAdj), kFinNorm, lam + i % kMaxPowerIters, nullptr, dscale_, nullptr);
    }
    check_cuda(cudaMemcpyAsync(hsc_, lam, lam_slots(power_iters) * 8, cudaMemcpyDeviceToHost, stream_),
               "D2H");
  } catch (...) {
    B_ = saveB;
    maps_.clear();
    throw;
  }
  B_ = saveB;
  maps_.clear();  // maps were encoded with zcount for batch 1
  estimate_pending_ = power_iters;
  estimate_f64_ = false;
}

double Plan::estimate_collect() {
  const size_t power_iters = estimate_pending_;
  if (power_iters == 0) fail(NDC_ERR_ARGUMENT, "estimate_collect without estimate_launch");
  estimate_pending_ = 0;
  if (estimate_f64_) return estimate_value_;
  sync();
  const double step = 1.0 / collect_lambdas(power_iters);
  // restore the per-image scale to 1 for later kEpiStore users
  std::vector<float> ones(B_, 1.0f);
  check_cuda(cudaMemcpyAsync(dscale_, ones.data(), B_ * 4, cudaMemcpyHostToDevice, stream_), "H2D");
  sync();
  return step;
}

// ---- NDTENSOR streaming (imageio.hpp:24-125 format) ----------------------------------------
namespace {
size_t first_nonfinite_serial(const double* v, size_t n) {
  for (size_t k = 0; k < n; ++k)
    if (!std::isfinite(v[k])) return k;
  return n;
}

struct Fd {
  int fd;
  ~Fd() {
    if (fd >= 0) ::close(fd);
  }
};

// Full-length pread / pwrite (they may transfer less than asked).
bool pread_all(int fd, void* buf, size_t n, size_t off) {
  char* p = static_cast<char*>(buf);
  while (n) {
    const ssize_t r = ::pread(fd, p, n, static_cast<off_t>(off));
    if (r <= 0) return false;
    p += r;
    off += static_cast<size_t>(r);
    n -= static_cast<size_t>(r);
  }
  return true;
}

bool pwrite_all(int fd, const void* buf, size_t n, size_t off) {
  const char* p = static_cast<const char*>(buf);
  while (n) {
    const ssize_t r = ::pwrite(fd, p, n, static_cast<off_t>(off));
    if (r <= 0) return false;
    p += r;
    off += static_cast<size_t>(r);
    n -= static_cast<size_t>(r);
  }
  return true;
}

// One pinned chunk of n doubles at file offset `off`, split over the host pool: each
// part is read (or written) and range-checked by its own thread.  Returns the first
// non-finite element (n if none); `io_ok` reports short reads / failed writes.
size_t chunk_io(bool write, int fd, double* buf, size_t n, size_t off, bool& io_ok) {
  HostPool& pool = HostPool::get();
  const unsigned parts = std::max(1u, std::min<unsigned>(pool.width(), static_cast<unsigned>(n >> 17)));
  std::vector<size_t> bad(parts, n);
  std::vector<char> ok(parts, 1);
  pool.run(parts, [&](unsigned i) {
    const auto r = part_range(n, parts, i);
    const size_t cnt = r.second - r.first;
    if (!write) ok[i] = pread_all(fd, buf + r.first, cnt * 8, off + r.first * 8);
    if (ok[i]) {
      const size_t k = first_nonfinite_serial(buf + r.first, cnt);
      if (k < cnt) bad[i] = r.first + k;
    }
    if (write && bad[i] == n) ok[i] = pwrite_all(fd, buf + r.first, cnt * 8, off + r.first * 8);
  });
  io_ok = std::all_of(ok.begin(), ok.end(), [](char c) { return c != 0; });
  return *std::min_element(bad.begin(), bad.end());
}
}  // namespace

std::vector<size_t> Plan::user_shape(bool y) const {
  std::vector<size_t> e;
  if (B_ > 1) e.push_back(B_);
  for (int i = 0; i < ndim_; ++i) e.push_back(y ? uext_x_[i] + uext_k_[i] - 1 : uext_x_[i]);
  return e;
}

// Streams the owned planes of an NDTENSOR file into HBM: each 16 MB pinned chunk is read
// and checked by the host pool while the previous chunk's H2D is in flight.
void Plan::load_observation_ndtensor(const std::string& path) {
  drain_halos();
  const NdtHeader h = read_ndtensor_header(path);
  if (h.ext != user_shape(true))
    fail(NDC_ERR_SHAPE, "load_observation: file shape does not match the plan's observation shape");
  ensure_pinned();
  Fd fd{::open(path.c_str(), O_RDONLY)};
  if (fd.fd < 0) fail(NDC_ERR_FORMAT, "cannot open " + path);
  const size_t plane = static_cast<size_t>(Y_.ey) * Y_.ex;                       // dense
  const size_t full = static_cast<size_t>(y_planes_total()) * plane;            // one image
  const size_t own = static_cast<size_t>(ny_user_planes_) * plane;
  const size_t chunk = kPinChunk / 8;
  size_t i = 0;
  for (size_t b = 0; b < B_; ++b) {
    const size_t first = b * full + static_cast<size_t>(ya_) * plane;
    for (size_t off = 0; off < own; off += chunk, ++i) {
      const int s = static_cast<int>(i & 1);
      const size_t n = std::min(chunk, own - off);
      check_cuda(cudaEventSynchronize(pin_ev_[s]), "cudaEventSynchronize");  // the slot's last DMA
      double* buf = static_cast<double*>(hpin_[s]);
      bool io_ok = true;
      const size_t bad = chunk_io(false, fd.fd, buf, n, h.payload_offset + (first + off) * 8, io_ok);
      if (!io_ok) fail(NDC_ERR_FORMAT, "read_tensor: truncated payload at element " + std::to_string(first + off));
      if (bad < n)
        fail(NDC_ERR_FORMAT, "read_tensor: non-finite value at element " + std::to_string(first + off + bad));
      check_cuda(cudaMemcpyAsync(static_cast<double*>(staging_) + off, buf, n * 8, cudaMemcpyHostToDevice,
                                 stream_),
                 "H2D");
      check_cuda(cudaEventRecord(pin_ev_[s], stream_), "cudaEventRecord");
    }
    check_cuda(launch_pack_f64(static_cast<const double*>(staging_),
                               yobs_ + b * Y_.image + static_cast<long long>(ya_ - rlo_) * Y_.plane, 1,
                               Y_.geo(ny_user_planes_), stream_),
               "pack");
    st_[2].launches++;
  }
  sync();
  halo_y(yobs_);
}

// Streams the owned estimate planes out: the D2H of chunk k+1 overlaps the host pool's
// check + pwrite of chunk k.  Sharded ranks write their own planes of one file.
void Plan::save_estimate_ndtensor(const std::string& path) {
  drain_halos();
  const std::vector<size_t> ext = user_shape(false);
  const std::string hl = ndtensor_header_line(ext);
  const size_t plane = static_cast<size_t>(my_) * mx_;
  const size_t full = static_cast<size_t>(nreal_x_);  // one image (a merged plan's real voxels)
  if (rank_ == 0) {  // header + full-size file, then every rank fills its planes
    Fd fd{::open(path.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644)};
    if (fd.fd < 0) fail(NDC_ERR_FORMAT, "cannot open " + path + " for writing");
    bool ok = pwrite_all(fd.fd, hl.data(), hl.size(), 0);
    ok = ok && ::ftruncate(fd.fd, static_cast<off_t>(hl.size() + full * B_ * 8)) == 0;
    if (!ok) fail(NDC_ERR_FORMAT, "write_tensor: stream failure");
  }
  if (world_ > 1) {  // barrier: the file exists before the other ranks open it
    comm_->allgather(dsc_, gather_, 1, stream_);
    sync();
  }
  ensure_pinned();
  Fd fd{::open(path.c_str(), O_WRONLY)};
  if (fd.fd < 0) fail(NDC_ERR_FORMAT, "cannot open " + path + " for writing");
  const size_t own = merged_ ? full : static_cast<size_t>(xa_n_) * plane;
  const size_t chunk = kPinChunk / 8;
  const size_t nchunks = (own + chunk - 1) / chunk;
  for (size_t b = 0; b < B_; ++b) {
    for (size_t r = 0; r < xruns_.size(); ++r) {  // one run unless merged
      check_cuda(launch_unpack_f64(x_owned(x_) + b * X_.image + static_cast<long long>(xruns_[r].first) * X_.plane,
                                   static_cast<double*>(staging_) + r * xrun_elems(), 1, X_.geo(xruns_[r].second),
                                   stream_),
                 "unpack");
      st_[2].launches++;
    }
    const size_t first = b * full + static_cast<size_t>(xa_) * plane;
    auto d2h = [&](size_t k) {
      const size_t n = std::min(chunk, own - k * chunk);
      check_cuda(cudaMemcpyAsync(hpin_[k & 1], static_cast<const double*>(staging_) + k * chunk, n * 8,
                                 cudaMemcpyDeviceToHost, stream_),
                 "D2H");
      check_cuda(cudaEventRecord(pin_ev_[k & 1], stream_), "cudaEventRecord");
    };
    d2h(0);
    for (size_t k = 0; k < nchunks; ++k) {
      if (k + 1 < nchunks) d2h(k + 1);
      check_cuda(cudaEventSynchronize(pin_ev_[k & 1]), "cudaEventSynchronize");
      const size_t n = std::min(chunk, own - k * chunk);
      bool io_ok = true;
      const size_t bad = chunk_io(true, fd.fd, static_cast<double*>(hpin_[k & 1]), n,
                                  hl.size() + (first + k * chunk) * 8, io_ok);
      if (bad < n) {
        sync();
        fail(NDC_ERR_NUMERIC, "write_tensor: refusing to store non-finite values");
      }
      if (!io_ok) {
        sync();
        fail(NDC_ERR_FORMAT, "write_tensor: stream failure");
      }
    }
  }
  if (world_ > 1) {  // every rank's planes are on disk before any returns
    comm_->allgather(dsc_, gather_, 1, stream_);
    sync();
  }
}

void Plan::add_gaussian_noise(double mean, double std_dev, uint64_t seed) {
  drain_halos();
  if (std_dev < 0) fail(NDC_ERR_NUMERIC, "add_gaussian_noise: std_dev must be >= 0");
  const size_t plane = static_cast<size_t>(Y_.ey) * Y_.ex;
  const size_t full = static_cast<size_t>(y_planes_total()) * plane;
  const size_t own = static_cast<size_t>(ny_user_planes_) * plane;
  double* dense = static_cast<double*>(staging_);
  GaussianNoise noise(seed, mean, std_dev, stream_);
  for (size_t b = 0; b < B_; ++b) {
    float* base = yobs_ + b * Y_.image + static_cast<long long>(ya_ - rlo_) * Y_.plane;
    check_cuda(launch_unpack_f64(base, dense, 1, Y_.geo(ny_user_planes_), stream_), "unpack");
    noise.add(dense, own, b * full + static_cast<size_t>(ya_) * plane);
    check_cuda(launch_pack_f64(dense, base, 1, Y_.geo(ny_user_planes_), stream_), "pack");
    st_[2].launches += 2;
  }
  sync();
  halo_y(yobs_);
}

// solvers.hpp:127-143 in float64 on dense scratch buffers (small problems only).
double Plan::estimate_step_f64(size_t power_iters) {
  const long long nx = static_cast<long long>(mz_) * my_ * mx_;
  const int oz = mz_ + 2 * pz_, oy = my_ + 2 * py_, ox = mx_ + 2 * px_;
  const long long ny = static_cast<long long>(oz) * oy * ox;
  const size_t K = h64_.size();
  std::vector<double> hf(h64_.rbegin(), h64_.rend());  // flip (kernel.hpp:41-45)
  double* dh = static_cast<double*>(dmalloc(K * 8));
  double* dhf = static_cast<double*>(dmalloc(K * 8));
  double* v = static_cast<double*>(dmalloc(nx * 8));
  double* u = static_cast<double*>(dmalloc(ny * 8));
  const long long nbx = (nx + 255) / 256;
  double2* part = static_cast<double2*>(dmalloc(nbx * sizeof(double2)));
  double* lam = dsc_ + kNumSlots * B_;
  struct Free {
    Plan* p;
    void* q[5];
    ~Free() {
      for (void* x : q) p->dfree(x);
    }
  } fr{this, {dh, dhf, v, u, part}};
  check_cuda(cudaMemcpyAsync(dh, h64_.data(), K * 8, cudaMemcpyHostToDevice, stream_), "H2D");
  check_cuda(cudaMemcpyAsync(dhf, hf.data(), K * 8, cudaMemcpyHostToDevice, stream_), "H2D");
  check_cuda(launch_fill_f64(v, 1.0 / std::sqrt(static_cast<double>(nx)), nx, stream_), "fill");
  st_[2].launches++;
  for (size_t i = 0; i < power_iters; ++i) {
    // u = A v_i with v_i = w_{i-1} / lambda_{i-1} folded in as an output scale
    long long nb = 0;
    check_cuda(launch_corr_f64(v, mz_, my_, mx_, u, oz, oy, ox, dhf, KZ_, KY_, KX_, -2 * pz_, -2 * py_,
                               -2 * px_, i ? lam + (i - 1) % kMaxPowerIters : nullptr, nullptr, &nb, stream_),
               "corr_f64 launch");
    // w = A^T u (valid correlation), ||w||^2 per block
    check_cuda(launch_corr_f64(u, oz, oy, ox, v, mz_, my_, mx_, dh, KZ_, KY_, KX_, 0, 0, 0, nullptr, part,
                               &nb, stream_),
               "corr_f64 launch");
    check_cuda(launch_finalize(part, nb, 1, kFinNorm, lam + i % kMaxPowerIters, nullptr, nullptr, nullptr,
                               stream_),
               "finalize launch");
    st_[2].launches += 3;
  }
  check_cuda(cudaMemcpyAsync(hsc_, lam, lam_slots(power_iters) * 8, cudaMemcpyDeviceToHost, stream_), "D2H");
  sync();
  return 1.0 / collect_lambdas(power_iters);
}

// The device power iterations record lambda_i in a ring of kMaxPowerIters slots (any
// power_iters is accepted, as in the reference).  A degenerate lambda (<= 0 or
// non-finite, solvers.hpp:137-139) makes the next rescale 1/lambda infinite or NaN, so
// every later lambda is NaN: checking the slots still held covers the whole run.
size_t Plan::lam_slots(size_t power_iters) {
  return std::min(power_iters, static_cast<size_t>(kMaxPowerIters));
}

double Plan::collect_lambdas(size_t power_iters) {
  for (size_t i = 0; i < lam_slots(power_iters); ++i)
    if (!(hsc_[i] > 0.0) || !std::isfinite(hsc_[i]))
      fail(NDC_ERR_NUMERIC, "estimate_step: degenerate convolution operator");
  return hsc_[(power_iters - 1) % kMaxPowerIters];
}

// estimate_step (solvers.hpp:127-143) for a separable PSF h[z][y][x] = a[z] b[y] c[x]:
// then A = A_z (x) A_y (x) A_x (Kronecker), the start vector ones/||ones|| is the Kronecker
// product of the 1-D normalised all-ones vectors, and A^T A maps Kronecker products to
// Kronecker products with ||w|| = prod_i ||w_i||.  So every iterate of the reference's
// power iteration is the Kronecker product of the 1-D iterates (each normalised by its own
// norm), and lambda_k = prod_i lambda_{i,k} -- the same sequence, computed in float64 on the
// host in O(power_iters * sum_i m_i k_i) instead of 2 * power_iters device passes.
// Rank-1 test: every entry of h against a[z] b[y] c[x] / h_max^2 (factors read through its
// largest entry) to 1e-6 of that entry -- separable Gaussians rounded to float32 (the
// BASELINE PSFs) pass it.  The iteration then runs on the rank-1 s with
// sum|h - s| <= 1e-6 sum|h|, so ||A_h - A_s|| <= 1e-6 ||h||_1 and the step moves by
// <= ~2e-6 relative (typically ~1e-7); the float32 device power iteration it replaces
// agrees with the reference to ~1e-5, and an exactly separable h reproduces the reference
// to rounding (tests/test_gpu_step.py).  Small problems keep the device float64 path
// (reference-exact on the tiny KATs); NDC_SEPARABLE_STEP=0 disables this path.
bool Plan::estimate_step_separable(size_t power_iters, double* step) {
  if (merged_) return false;  // the merged plane axis carries zero planes: not a Kronecker product
  if (const char* e = std::getenv("NDC_SEPARABLE_STEP"))
    if (std::atoi(e) == 0) return false;
  if (h64_.empty()) return false;
  const int k[3] = {KZ_, KY_, KX_};
  const int m[3] = {mz_, my_, mx_};
  size_t imax = 0;
  for (size_t i = 1; i < h64_.size(); ++i)
    if (std::fabs(h64_[i]) > std::fabs(h64_[imax])) imax = i;
  const double hmax = h64_[imax];
  if (!(std::fabs(hmax) > 0.0) || !std::isfinite(hmax)) return false;
  const int i0 = static_cast<int>(imax / (static_cast<size_t>(KY_) * KX_));
  const int j0 = static_cast<int>((imax / KX_) % KY_);
  const int l0 = static_cast<int>(imax % KX_);
  auto at = [&](int z, int y, int x) { return h64_[(static_cast<size_t>(z) * KY_ + y) * KX_ + x]; };
  std::vector<double> f[3];
  for (int z = 0; z < KZ_; ++z) f[0].push_back(at(z, j0, l0));
  for (int y = 0; y < KY_; ++y) f[1].push_back(at(i0, y, l0));
  for (int x = 0; x < KX_; ++x) f[2].push_back(at(i0, j0, x) / (hmax * hmax));
  for (int z = 0; z < KZ_; ++z)
    for (int y = 0; y < KY_; ++y)
      for (int x = 0; x < KX_; ++x) {
        const double hv = at(z, y, x);
        if (!(std::fabs(hv - f[0][z] * f[1][y] * f[2][x]) <= 1e-6 * std::fabs(hv))) return false;
      }
  std::vector<double> lam(power_iters, 1.0);
  for (int d = 0; d < 3; ++d) {
    const int n = m[d], kk = k[d];
    std::vector<double> v(n, 1.0 / std::sqrt(static_cast<double>(n))), u(n + kk - 1), w(n);
    for (size_t it = 0; it < power_iters; ++it) {
      // u = conv_full(v, f): u[s] = sum_j f[j] v[s - j]
      for (int s2 = 0; s2 < n + kk - 1; ++s2) {
        double acc = 0.0;
        for (int j = std::max(0, s2 - n + 1); j <= std::min(kk - 1, s2); ++j) acc += f[d][j] * v[s2 - j];
        u[s2] = acc;
      }
      // w = A^T u: valid correlation w[t] = sum_j f[j] u[t + j]
      double nrm = 0.0;
      for (int t = 0; t < n; ++t) {
        double acc = 0.0;
        for (int j = 0; j < kk; ++j) acc += f[d][j] * u[t + j];
        w[t] = acc;
        nrm += acc * acc;
      }
      nrm = std::sqrt(nrm);
      lam[it] *= nrm;
      if (!(nrm > 0.0) || !std::isfinite(nrm)) {
        lam[it] = nrm;  // degenerate: reported below like the reference
        break;
      }
      for (int t = 0; t < n; ++t) v[t] = w[t] / nrm;
    }
  }
  for (size_t it = 0; it < power_iters; ++it)
    if (!(lam[it] > 0.0) || !std::isfinite(lam[it]))
      fail(NDC_ERR_NUMERIC, "estimate_step: degenerate convolution operator");
  *step = 1.0 / lam[power_iters - 1];
  return true;
}

// ---- projected gradient ---------------------------------------------------------------
void Plan::pg_begin(const ndc_deconv_config& c) {
  // solvers.hpp:65-76
  if (c.max_iters == 0) fail(NDC_ERR_CONFIG, "DeconvConfig: max_iters must be positive");
  if (!(c.tol_rel_objective >= 0)) fail(NDC_ERR_CONFIG, "DeconvConfig: tol_rel_objective must be >= 0");
  if (c.has_initial_step && !(c.initial_step > 0))
    fail(NDC_ERR_CONFIG, "DeconvConfig: initial_step must be positive");
  if (!(c.backtrack_factor > 0) || !(c.backtrack_factor < 1))
    fail(NDC_ERR_CONFIG, "DeconvConfig: backtrack_factor must be in (0,1)");
  if (c.max_backtracks == 0) fail(NDC_ERR_CONFIG, "DeconvConfig: max_backtracks must be positive");
  if (c.power_iters == 0) fail(NDC_ERR_CONFIG, "DeconvConfig: power_iters must be positive");
  if (kernel_all_zero_) fail(NDC_ERR_NUMERIC, "deconv_pg: degenerate all-zero kernel");
  cfg_ = c;
  wall0_ = now_s();
  step0_ = c.has_initial_step ? c.initial_step : estimate_step(c.power_iters);

  img_.assign(B_, Img{});
  std::vector<int> act(B_, 1);
  upload_active(act);
  // x0 = max(A^T y, 0) (solvers.hpp:166-167); A x0 and f (168-172)
  correlate(kAdj, yobs_, x_, kEpiClamp, nullptr, nullptr, nullptr, nullptr, nullptr, false);
  halo_x(x_);
  correlate(kFwd, x_, r_, kEpiResid, nullptr, yobs_, nullptr, nullptr, nullptr, true);
  finalize(partials_per_image(kFwd), kFinHalfSum, dsc_ + kF * B_, nullptr, nullptr, nullptr);
  check_cuda(cudaMemcpyAsync(hsc_, dsc_ + kF * B_, B_ * 8, cudaMemcpyDeviceToHost, stream_), "D2H");
  std::vector<double> steps(B_, step0_);
  upload_steps(steps);
  sync();
  for (size_t b = 0; b < B_; ++b) {
    img_[b].f = hsc_[b];
    img_[b].obj.push_back(hsc_[b]);
    img_[b].step = step0_;
  }
  halo_y(r_);
  spec_ready_ = false;
  pg_begun_ = true;
}

// One PG iteration per step, per image (solvers.hpp:179-228).  Common case -- every
// active image accepts its first trial -- runs speculatively ahead: right after the
// forward pass and the scalar read-back of step k are enqueued, the adjoint of step k+1
// is enqueued too (as if every trial is accepted: r = r_trial, x = trial, into spare
// buffers), so the device keeps working while the host makes step k's decision.  When
// every image did accept (and none stops), the buffers rotate and step k+1 starts at
// its forward pass; otherwise the speculative pass is discarded (its inputs are
// unchanged, so it is exact when kept).  z-slab ranks take identical decisions, so they
// speculate identically.
size_t Plan::pg_iterate(size_t n) {
  if (!pg_begun_) fail(NDC_ERR_ARGUMENT, "pg_iterate before pg_begin");
  static const bool spec_on = [] {
    const char* e = std::getenv("NDC_SPECULATE");
    return e == nullptr || std::atoi(e) != 0;
  }();
  size_t active_count = 0;
  for (size_t step = 0; step < n; ++step) {
    std::vector<int> act(B_, 0);
    active_count = 0;
    for (size_t b = 0; b < B_; ++b) {
      Img& im = img_[b];
      if (im.active && im.kkt.size() >= cfg_.max_iters) im.active = false;  // max_iters
      act[b] = im.active ? 1 : 0;
      active_count += act[b];
    }
    if (active_count == 0) break;
    if (spec_ready_ && act != act_cache_) spec_ready_ = false;  // the set changed: recompute
    upload_active(act);
    upload_steps(std::vector<double>(B_, step0_));

    if (!spec_ready_) {
      // g = A^T(A x - y) with kkt, trial = max(x - step0 g, 0), changed count (180-191)
      correlate(kAdj, r_, trial_, kEpiPG, g_, x_, nullptr, dstep_, dactive_, true);
      halo_x(trial_);  // z-slabs: overlaps the forward pass's interior planes
      finalize(partials_per_image(kAdj), kFinMaxSum, dsc_ + kKKT * B_, dsc_ + kCHG * B_, nullptr,
               dactive_);
    }
    spec_ready_ = false;
    // A trial, residual, f_trial (195-197)
    correlate(kFwd, trial_, rt_, kEpiResid, nullptr, yobs_, nullptr, nullptr, dactive_, true);
    halo_y(rt_);  // z-slabs: r_trial's halo, needed by the next adjoint if it is accepted
    finalize(partials_per_image(kFwd), kFinHalfSum, dsc_ + kAUX * B_, nullptr, nullptr, dactive_);
    check_cuda(cudaMemcpyAsync(hsc_, dsc_, kNumSlots * B_ * 8, cudaMemcpyDeviceToHost, stream_), "D2H");
    check_cuda(cudaEventRecord(d2h_ev_, stream_), "cudaEventRecord");

    // speculative adjoint of the next step (see above); needs a next step for every image
    bool spec = spec_on;
    for (size_t b = 0; b < B_ && spec; ++b)
      if (act[b] && img_[b].kkt.size() + 1 >= cfg_.max_iters) spec = false;
    if (spec) {
      if (!trial2_) {
        const long long nx = X_.image * static_cast<long long>(B_);
        trial2_ = dev_alloc_f(nx);
        g2_ = dev_alloc_f(nx);
      }
      correlate(kAdj, rt_, trial2_, kEpiPG, g2_, trial_, nullptr, dstep_, dactive_, true);
      halo_x(trial2_);
      finalize(partials_per_image(kAdj), kFinMaxSum, dsc_ + kKKT * B_, dsc_ + kCHG * B_, nullptr, dactive_);
    }
    check_cuda(cudaEventSynchronize(d2h_ev_), "cudaEventSynchronize");

    // per-image decision (191-205)
    enum { kAccept, kFixed, kBacktrack, kStall };
    std::vector<int> state(B_, -1);
    std::vector<double> ft(B_, 0.0), stp(B_, step0_);
    std::vector<size_t> nbt(B_, 0);
    for (size_t b = 0; b < B_; ++b) {
      if (!act[b]) continue;
      img_[b].kkt.push_back(hsc_[kKKT * B_ + b]);
      const double chg = hsc_[kCHG * B_ + b];
      ft[b] = hsc_[kAUX * B_ + b];
      if (chg == 0.0)
        state[b] = kFixed;
      else if (ft[b] < img_[b].f)
        state[b] = kAccept;
      else
        state[b] = kBacktrack;
    }
    bool all_accept = true;
    for (size_t b = 0; b < B_; ++b)
      if (act[b] && state[b] != kAccept) all_accept = false;
    // backtracking: step *= factor, up to max_backtracks more trials (189, 205)
    for (;;) {
      std::vector<int> bt(B_, 0);
      size_t nb = 0;
      for (size_t b = 0; b < B_; ++b) {
        if (state[b] != kBacktrack) continue;
        if (nbt[b] + 1 > cfg_.max_backtracks) {
          state[b] = kStall;
          continue;
        }
        nbt[b]++;
        img_[b].backtracks++;
        stp[b] *= cfg_.backtrack_factor;
        bt[b] = 1;
        nb++;
      }
      if (nb == 0) break;
      upload_active(bt);
      upload_steps(stp);
      drain_halos();  // trial_ is rewritten outside correlate()
      check_cuda(launch_pg_trial(x_owned(x_), x_owned(g_), x_owned(trial_), dstep_, dactive_, partials_,
                                 static_cast<int>(B_), X_.geo(xa_n_), kElemBlocks, stream_),
                 "pg_trial launch");
      st_[2].launches++;
      finalize(kElemBlocks, kFinSumSum, dsc_ + kAUX * B_, dsc_ + kCHG * B_, nullptr, dactive_);
      halo_x(trial_);
      correlate(kFwd, trial_, rt_, kEpiResid, nullptr, yobs_, nullptr, nullptr, dactive_, true);
      halo_y(rt_);
      finalize(partials_per_image(kFwd), kFinHalfSum, dsc_ + kAUX * B_, nullptr, nullptr, dactive_);
      check_cuda(cudaMemcpyAsync(hsc_, dsc_, kNumSlots * B_ * 8, cudaMemcpyDeviceToHost, stream_),
                 "D2H");
      sync();
      for (size_t b = 0; b < B_; ++b) {
        if (!bt[b]) continue;
        ft[b] = hsc_[kAUX * B_ + b];
        if (hsc_[kCHG * B_ + b] == 0.0)
          state[b] = kFixed;
        else if (ft[b] < img_[b].f)
          state[b] = kAccept;
      }
    }
    // commit (208-227)
    bool any_accept = false, any_stop = false;
    for (size_t b = 0; b < B_; ++b) {
      if (!act[b]) continue;
      Img& im = img_[b];
      if (state[b] == kFixed) {
        im.reason = NDC_STOP_CONVERGED;
        im.active = false;
        any_stop = true;
      } else if (state[b] == kStall) {
        im.reason = NDC_STOP_STALLED;
        im.active = false;
        any_stop = true;
      } else {
        any_accept = true;
        const double drop = im.f - ft[b];
        im.f = ft[b];
        im.obj.push_back(ft[b]);
        im.iters = im.kkt.size();
        if (drop <= cfg_.tol_rel_objective * im.obj[im.obj.size() - 2]) {
          im.reason = NDC_STOP_CONVERGED;
          im.active = false;
          any_stop = true;
        }
      }
    }
    if (spec && all_accept && !any_stop) {
      // keep the speculative adjoint: x <- trial, r <- r_trial, and the next step's
      // trial / g are already in trial2 / g2
      float* old_x = x_;
      x_ = trial_;
      trial_ = trial2_;
      trial2_ = old_x;
      std::swap(g_, g2_);
      std::swap(r_, rt_);
      // Images that stopped at an earlier step were skipped by both passes: the rotated
      // x / r buffers hold stale data for them, so their last iterate and residual are
      // copied back (pg_end's final KKT and the estimate read them).
      for (size_t b = 0; b < B_; ++b)
        if (!act[b]) {
          copy_image_x(x_, old_x, b);
          copy_image_y(r_, rt_, b);
        }
      spec_ready_ = true;
      continue;
    }
    if (any_accept) {
      std::swap(x_, trial_);
      std::swap(r_, rt_);
      // images that did not accept (stopped now or earlier) keep their previous iterate
      for (size_t b = 0; b < B_; ++b)
        if (state[b] != kAccept) {
          copy_image_x(x_, trial_, b);
          copy_image_y(r_, rt_, b);  // with its halo planes
        }
    }
  }
  active_count = 0;
  for (auto& im : img_)
    if (im.active && im.kkt.size() < cfg_.max_iters) active_count++;
  return active_count;
}

// Fill image b's real x planes (a merged plan's zero planes stay zero).
void Plan::fill_x_real(float* buf, size_t b, float v) {
  for (const auto& r : xruns_) {
    check_cuda(launch_fill(x_owned(buf) + b * X_.image + static_cast<long long>(r.first) * X_.plane, v, 1,
                           X_.geo(r.second), stream_),
               "fill");
    st_[2].launches++;
  }
}

void Plan::copy_image_x(float* dst, const float* src, size_t b) {
  drain_halos();
  check_cuda(cudaMemcpyAsync(dst + b * X_.image, src + b * X_.image, X_.image * 4,
                             cudaMemcpyDeviceToDevice, stream_),
             "D2D");
}
void Plan::copy_image_y(float* dst, const float* src, size_t b) {
  drain_halos();
  check_cuda(cudaMemcpyAsync(dst + b * Y_.image, src + b * Y_.image, Y_.image * 4,
                             cudaMemcpyDeviceToDevice, stream_),
             "D2D");
}

void Plan::pg_end() {
  if (!pg_begun_) fail(NDC_ERR_ARGUMENT, "pg_end before pg_begin");
  spec_ready_ = false;  // a speculative next-step adjoint, if any, is simply dropped
  // solvers.hpp:230-233: one more adjoint for images whose last iterate has no KKT.
  std::vector<int> need(B_, 0);
  size_t nneed = 0;
  for (size_t b = 0; b < B_; ++b)
    if (img_[b].kkt.size() < img_[b].obj.size()) {
      need[b] = 1;
      nneed++;
    }
  if (nneed) {
    upload_active(need);
    correlate(kAdj, r_, nullptr, kEpiKKT, nullptr, x_, nullptr, nullptr, dactive_, true);
    finalize(partials_per_image(kAdj), kFinMaxSum, dsc_ + kKKT * B_, dsc_ + kCHG * B_, nullptr,
             dactive_);
    check_cuda(cudaMemcpyAsync(hsc_, dsc_, kNumSlots * B_ * 8, cudaMemcpyDeviceToHost, stream_), "D2H");
    sync();
    for (size_t b = 0; b < B_; ++b)
      if (need[b]) img_[b].kkt.push_back(hsc_[kKKT * B_ + b]);
  }
  std::vector<int> all(B_, 1);
  upload_active(all);
  wall_ = now_s() - wall0_;
  pg_begun_ = false;
}

void Plan::get_report(size_t image, ndc_deconv_report* rep, double* obj, double* kkt,
                      size_t cap) const {
  if (image >= img_.size()) fail(NDC_ERR_ARGUMENT, "report: image index out of range");
  const Img& im = img_[image];
  if (cap < im.obj.size() || cap < im.kkt.size())
    fail(NDC_ERR_ARGUMENT, "report: trace capacity too small");
  rep->iterations_run = im.iters;
  rep->stop_reason = im.reason;
  rep->wall_time_seconds = wall_;
  rep->negative_pixels_clamped = im.clamped;
  rep->trace_len = im.obj.size();
  rep->backtracks = im.backtracks;
  rep->step0 = step0_;
  if (obj) std::memcpy(obj, im.obj.data(), im.obj.size() * 8);
  if (kkt) std::memcpy(kkt, im.kkt.data(), im.kkt.size() * 8);
}

void Plan::bench_forward() {
  correlate(kFwd, x_, rt_, kEpiResid, nullptr, yobs_, nullptr, nullptr, nullptr, true);
}
void Plan::bench_adjoint() {
  correlate(kAdj, r_, trial_, kEpiPG, g_, x_, nullptr, dstep_, nullptr, true);
}

// ---- Richardson-Lucy (solvers.hpp:245-305) ----------------------------------------------
// Taps: adjoint correlates with h, forward with flip(h) (kernel.hpp:41-45); each
// (kz, ky) row stored with the even pitch tap_pitch(KX) (zero pad).
void Plan::set_taps(double scale) {
  const size_t count = h64_.size();
  const int kxp = tap_pitch(KX_);
  const size_t rows = count / KX_;
  taps_adj_.assign(rows * kxp, 0.0f);
  taps_fwd_.assign(rows * kxp, 0.0f);
  for (size_t i = 0; i < count; ++i) {
    const size_t j = count - 1 - i;  // flipped flat index
    const float v = static_cast<float>(scale == 1.0 ? h64_[i] : h64_[i] * scale);
    taps_adj_[(i / KX_) * kxp + i % KX_] = v;
    taps_fwd_[(j / KX_) * kxp + j % KX_] = v;
  }
  chunks_fwd_ = build_chunks(taps_fwd_);
  chunks_adj_ = build_chunks(taps_adj_);
}

// Tap chunks of one direction: columns [kx0, kx0 + cw) (instantiation width w >= cw, zero
// padded), rows [ky0, ky0 + cy), z-slices [kz0, kz1).  One chunk for every PSF up to 33
// columns, kcy_ rows and kTapCap taps (all BASELINE configs but config 5, which splits
// in z).  z-slices whose taps are all zero are skipped (they add exact zeros): the merged
// plane axis of a tensor with more than 3 dimensions is mostly such slices.
std::vector<TapChunk> Plan::build_chunks(const std::vector<float>& taps) const {
  const int kxp = tap_pitch(KX_);
  const size_t slice = static_cast<size_t>(KY_) * kxp;
  std::vector<std::pair<int, int>> zruns;  // maximal runs of slices with a nonzero tap
  for (int kz = 0; kz < KZ_;) {
    const bool nz = std::any_of(taps.begin() + kz * slice, taps.begin() + (kz + 1) * slice,
                                [](float v) { return v != 0.0f; });
    if (!nz) {
      ++kz;
      continue;
    }
    int e = kz + 1;
    while (e < KZ_ && std::any_of(taps.begin() + e * slice, taps.begin() + (e + 1) * slice,
                                  [](float v) { return v != 0.0f; }))
      ++e;
    zruns.push_back({kz, e});
    kz = e;
  }
  if (zruns.empty()) zruns.push_back({0, KZ_});  // an all-zero kernel still runs (zero output)
  std::vector<TapChunk> chunks;
  for (int kx0 = 0; kx0 < KX_; kx0 += (KX_ <= kMaxKX ? KX_ : kMaxKX - 1)) {
    const int cw = KX_ <= kMaxKX ? KX_ : std::min(kMaxKX - 1, KX_ - kx0);
    const int w = (cw % 2) ? cw : cw + 1;
    for (int ky0 = 0; ky0 < KY_; ky0 += kcy_) {
      const int cy = std::min(kcy_, KY_ - ky0);
      const int slices = std::max(1, kTapCap / (cy * tap_pitch(w)));
      for (const auto& zr : zruns)
        for (int kz0 = zr.first; kz0 < zr.second; kz0 += slices)
          chunks.push_back({kx0, cw, w, ky0, cy, kz0, std::min(zr.second, kz0 + slices)});
    }
  }
  return chunks;
}

// Richardson-Lucy (solvers.hpp:245-305) on the same operators: the kernel normalised to
// unit sum, negative observations clamped (and counted), x0 = sum(yc)/n, then
//   ratio = guarded_div(yc, A x)        forward pass, fused with r = Ax - yc, 0.5||r||^2
//   kkt   = max|min(x, A^T r)|          adjoint pass (record, solvers.hpp:284-289)
//   x'    = x .* A^T ratio, ||x'-x||, ||x||   adjoint pass (290-292)
// per image, one 3-scalar D2H per iteration.
void Plan::rl_run(const ndc_rl_config& c) {
  drain_halos();
  if (c.max_iters == 0) fail(NDC_ERR_CONFIG, "RlConfig: max_iters must be positive");
  if (!(c.tol_rel_change >= 0)) fail(NDC_ERR_CONFIG, "RlConfig: tol_rel_change must be >= 0");
  double hsum = 0.0;
  for (double v : h64_) {
    if (v < 0.0) fail(NDC_ERR_NUMERIC, "deconv_rl: kernel entries must be nonnegative");
    hsum += v;
  }
  if (!(hsum > 0.0)) fail(NDC_ERR_NUMERIC, "deconv_rl: kernel must have positive sum");
  wall0_ = now_s();
  // hn = scale(h, 1/hsum) (solvers.hpp:256): multiply in f64 as the reference does
  {
    std::vector<double> hn(h64_.size());
    for (size_t i = 0; i < hn.size(); ++i) hn[i] = h64_[i] * (1.0 / hsum);
    std::swap(hn, h64_);
    set_taps(1.0);
    std::swap(hn, h64_);
  }
  // yc = clamp(y) goes to a y-shaped buffer of its own for the run (the reference's
  // deconv_rl leaves y untouched: the resident observation stays the user's data)
  float* const y_user = yobs_;
  float* const yc = dev_alloc_f(Y_.image * static_cast<long long>(B_));
  struct Restore {
    Plan* p;
    float* y_user;
    float* yc;
    ~Restore() {
      p->drain_halos();
      p->yobs_ = y_user;
      p->dfree(yc);
      p->set_taps(1.0);
    }
  } restore{this, y_user, yc};

  img_.assign(B_, Img{});
  // yc = clamp(y), negatives counted, total = sum(yc)
  const Geo yv = Y_.geo(yb_ - ya_);
  const long long own_off = static_cast<long long>(ya_ - rlo_) * Y_.plane;
  check_cuda(launch_clamp_count(y_user + own_off, yc + own_off, partials_, static_cast<int>(B_), yv,
                                kElemBlocks, stream_),
             "clamp launch");
  yobs_ = yc;  // the RL passes below read the clamped copy
  st_[2].launches++;
  finalize(kElemBlocks, kFinSumSum, dsc_ + kAUX * B_, dsc_ + kCHG * B_, nullptr, nullptr);
  check_cuda(cudaMemcpyAsync(hsc_, dsc_, kNumSlots * B_ * 8, cudaMemcpyDeviceToHost, stream_), "D2H");
  sync();
  halo_y(yobs_);
  std::vector<double> total(B_);
  std::vector<int> act(B_, 1);
  const double n = nreal_x_;
  for (size_t b = 0; b < B_; ++b) {
    total[b] = hsc_[kAUX * B_ + b];
    img_[b].clamped = static_cast<size_t>(hsc_[kCHG * B_ + b]);
  }
  // x0 per image: total/n, or 0 for an all-zero observation (solvers.hpp:263-270)
  for (size_t b = 0; b < B_; ++b) {
    const float v = total[b] > 0.0 ? static_cast<float>(total[b] / n) : 0.0f;
    fill_x_real(x_, b, v);
  }
  halo_x(x_);

  auto record = [&](const std::vector<int>& a) {
    // forward: ratio -> rt_, r -> r_, 0.5||r||^2 ; adjoint: kkt of x vs A^T r
    upload_active(a);
    correlate(kFwd, x_, rt_, kEpiRLRatio, r_, yobs_, nullptr, nullptr, dactive_, true);
    finalize(partials_per_image(kFwd), kFinHalfSum, dsc_ + kF * B_, nullptr, nullptr, dactive_);
    halo_y(r_);
    halo_y(rt_);
    correlate(kAdj, r_, nullptr, kEpiKKT, nullptr, x_, nullptr, nullptr, dactive_, true);
    finalize(partials_per_image(kAdj), kFinMaxSum, dsc_ + kKKT * B_, dsc_ + kCHG * B_, nullptr,
             dactive_);
    check_cuda(cudaMemcpyAsync(hsc_, dsc_, kNumSlots * B_ * 8, cudaMemcpyDeviceToHost, stream_), "D2H");
    sync();
    for (size_t b = 0; b < B_; ++b)
      if (a[b]) {
        img_[b].obj.push_back(hsc_[kF * B_ + b]);
        img_[b].kkt.push_back(hsc_[kKKT * B_ + b]);
      }
  };
  record(act);
  for (size_t b = 0; b < B_; ++b)
    if (!(total[b] > 0.0)) {
      img_[b].reason = NDC_STOP_CONVERGED;
      img_[b].active = false;
      act[b] = 0;
    }
  for (size_t k = 1; k <= c.max_iters; ++k) {
    size_t nact = 0;
    for (size_t b = 0; b < B_; ++b) nact += act[b];
    if (nact == 0) break;
    upload_active(act);
    // x' = x .* A^T ratio  (+ ||x'-x||^2, ||x||^2)
    correlate(kAdj, rt_, trial_, kEpiRLUpdate, nullptr, x_, nullptr, nullptr, dactive_, true);
    finalize(partials_per_image(kAdj), kFinSumSum, dsc_ + kAUX * B_, dsc_ + kCHG * B_, nullptr,
             dactive_);
    check_cuda(cudaMemcpyAsync(hsc_, dsc_, kNumSlots * B_ * 8, cudaMemcpyDeviceToHost, stream_), "D2H");
    sync();
    std::vector<double> rel(B_, 0.0);
    for (size_t b = 0; b < B_; ++b)
      if (act[b])
        rel[b] = std::sqrt(hsc_[kAUX * B_ + b]) / std::max(std::sqrt(hsc_[kCHG * B_ + b]), 1e-300);
    std::swap(x_, trial_);
    for (size_t b = 0; b < B_; ++b)
      if (!act[b]) copy_image_x(x_, trial_, b);  // stopped images keep their iterate
    halo_x(x_);
    record(act);
    for (size_t b = 0; b < B_; ++b) {
      if (!act[b]) continue;
      img_[b].iters = k;
      if (rel[b] < c.tol_rel_change) {
        img_[b].reason = NDC_STOP_CONVERGED;
        img_[b].active = false;
        act[b] = 0;
      }
    }
  }
  std::vector<int> all(B_, 1);
  upload_active(all);
  step0_ = 0.0;
  wall_ = now_s() - wall0_;
}

}  // namespace ndc

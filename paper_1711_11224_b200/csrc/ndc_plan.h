// Plan: device buffers, operators and the projected-gradient driver for one
// (x shape, kernel, batch) problem on one GPU -- or one z-slab of it on one rank.
//
// Mirrors ndconv::deconv_pg (solvers.hpp:155-238) with all tensors resident in HBM.
// Per iteration and image the host sees only a handful of f64 scalars (objective,
// KKT, changed-count) read back in one small D2H; the accept / backtrack / stop logic
// is the reference's, evaluated per image.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <set>
#include <memory>
#include <string>
#include <vector>

#include "ndc_internal.h"
#include "../../include/ndconv_b200.h"

namespace ndc {

struct Error {
  int code;
  std::string msg;
};
[[noreturn]] void fail(int code, const std::string& msg);
void check_cuda(cudaError_t e, const char* what);

// Pitched volume geometry of one image held locally.  x-shaped volumes carry a zero
// margin of r0 rows above and c0 (>= 2p_x, multiple of 4) columns left of the data so
// that every forward-pass TMA box starts at a non-negative coordinate (a negative
// tile start traps on this driver); `origin` is the offset of element (0,0,0).
struct Vol {
  int ez = 1, ey = 1, ex = 1;
  int r0 = 0, c0 = 0;
  long long pitch = 0, plane = 0, image = 0, origin = 0;
  static Vol make(int z, int y, int x, int r0 = 0, int c0 = 0);
  Geo geo(int nz) const { return Geo{nz, ey, ex, pitch, plane, image}; }
};

// Halo / scalar transport between z-slab ranks (null for an unsharded plan).
class Transport {
 public:
  virtual ~Transport() = default;
  virtual int rank() const = 0;
  virtual int world() const = 0;
  // Send `count` floats at send_lo to rank-1 and at send_hi to rank+1; receive into
  // recv_lo from rank-1 and recv_hi from rank+1 (null pointers skip a side).
  virtual void exchange(const float* send_lo, float* recv_lo, const float* send_hi, float* recv_hi,
                        size_t count, cudaStream_t s) = 0;
  // All-gather `n` doubles per rank: out[r*n + i] = rank r's in[i].
  virtual void allgather(const double* in, double* out, size_t n, cudaStream_t s) = 0;
};
std::unique_ptr<Transport> make_nccl_transport(int device, int rank, int world,
                                               const unsigned char id[128]);
struct LocalGroup;
LocalGroup* new_local_group(int world);
void delete_local_group(LocalGroup* g);
std::unique_ptr<Transport> make_local_transport(LocalGroup* g, int rank);
void nccl_unique_id(unsigned char out[128]);
double probe_fp32_peak(int device);  // measured FP32 FMA TFLOP/s (ndc_probe.cu)
unsigned long long guard_violations();  // guard bytes found changed so far (process-wide)

// One launch's share of the taps (see Plan::build_chunks).
struct TapChunk {
  int kx0, cw, w, ky0, cy, kz0, kz1;
};

struct KernelStats {
  uint64_t launches = 0;
  double ms = 0.0;
};

class Plan {
 public:
  Plan(int device, size_t batch, int ndim, const size_t* x_ext, const size_t* k_ext, const double* h,
       std::unique_ptr<Transport> comm = nullptr);
  ~Plan();
  Plan(const Plan&) = delete;
  Plan& operator=(const Plan&) = delete;

  // --- data movement (dense host arrays, owned planes only when sharded) ---
  void set_observation_f64(const double* y);
  void set_observation_f32(const float* y);
  void set_x_f64(const double* x);               // into the x buffer (for conv_full etc.)
  void set_x_f32(const float* x);
  void get_estimate_f64(double* x);
  void get_estimate_f32(float* x);
  void get_observation_f64(double* y);           // the resident (f32) observation
  void get_y_buffer_f64(double* y);              // the y-shaped result buffer (A x)
  void get_y_buffer_f32(float* y);
  void get_x_buffer_f32(float* x);
  void get_x_buffer_f64(double* x, int which);   // 0 = x, 1 = g
  void load_observation_ndtensor(const std::string& path);  // streamed, owned planes
  void save_estimate_ndtensor(const std::string& path);
  // add_gaussian_noise (simulation.hpp:184-191) to the resident observation in place, the
  // mt19937_64 stream running over the user's dense [batch, y...] storage order
  void add_gaussian_noise(double mean, double std_dev, uint64_t seed);
  std::vector<size_t> user_shape(bool y) const;   // [batch,] extents as the caller sees them

  // --- operators on resident buffers (the one-shot C-ABI entry points use these) ---
  void op_conv_full();                 // r = A x            (store)
  void op_adjoint_of_y();              // x = A^T y          (store)
  double op_objective();               // 0.5||A x - y||^2   (resid into r)
  void op_normal_gradient();           // g = A^T (A x - y)
  double op_kkt_residual();            // max|min(x, A^T(Ax - y))|
  double estimate_step(size_t power_iters);
  void estimate_launch(size_t power_iters);  // enqueue only (see ndc_plan.cu)
  bool kernel_all_zero() const { return kernel_all_zero_; }
  double estimate_collect();
  static size_t lam_slots(size_t power_iters);
  double collect_lambdas(size_t power_iters);
  double estimate_step_f64(size_t power_iters);  // small problems (reference-exact)
  // separable PSFs: the power iteration as a product of 1-D iterations (host, f64);
  // false if h is not rank-1
  bool estimate_step_separable(size_t power_iters, double* step);

  // --- projected gradient (solvers.hpp:155-238) ---
  void pg_begin(const ndc_deconv_config& cfg);
  size_t pg_iterate(size_t n);  // returns images still active
  void pg_end();
  void get_report(size_t image, ndc_deconv_report* rep, double* obj, double* kkt, size_t cap) const;

  // --- Richardson-Lucy (solvers.hpp:245-305) ---
  void rl_run(const ndc_rl_config& cfg);

  // --- debugging: guard-band mode (NDC_GUARD_BANDS=1) ---
  size_t check_guards();  // changed guard bytes around this plan's allocations (0 if off)
  void debug_corrupt_guard();  // the checker's own test: writes 16 bytes into a guard

  // --- bench hooks ---
  void set_timing(bool on) { timing_ = on; }
  void reset_stats();
  KernelStats stats(int kind);
  cudaStream_t stream() const { return stream_; }
  void bench_forward();
  void bench_adjoint();

  size_t batch() const { return B_; }
  size_t x_count() const { return xruns_.size() * xrun_elems(); }  // owned, per image
  size_t y_count() const { return static_cast<size_t>(ny_user_planes_) * (my_ + 2 * py_) * (mx_ + 2 * px_); }

 private:
  enum Dir { kFwd = 0, kAdj = 1 };
  void alloc_all();
  void* dmalloc(size_t bytes);
  void dfree(void* p);
  std::map<void*, std::pair<void*, size_t>> allocs_;  // guard-band mode: user -> (base, bytes)
  float* dev_alloc_f(long long n);
  void ensure_pinned();
  void release_pinned();
  void h2d_staged(void* dev, const void* host, size_t bytes);
  void d2h_staged(void* host, const void* dev, size_t bytes);
  void* hpin_[2] = {nullptr, nullptr};      // pinned staging ring (16 MB slots)
  cudaEvent_t pin_ev_[2] = {nullptr, nullptr};
  const CUtensorMap& map_for(const float* base, Dir d, int sh, int kx, int ky);
  // Correlation pass over resident buffers; mode / aux per EpiMode.
  void correlate(Dir d, const float* in, float* out, int mode, float* aux_out, const float* aux_in,
                 const float* scale, const double* step, const int* active, bool partials);
  // Reductions of the last correlate/elementwise pass into per-image device scalars.
  void finalize(long long per_image, int op, double* out0, double* out1, float* scale_out,
                const int* active);
  long long partials_per_image(Dir d) const;
  void halo_x(float* buf);   // fill x-buffer halo planes from neighbours (sharded only)
  void halo_y(float* buf);   // fill y-buffer halo planes from neighbours (sharded only)
  void halo_enqueue(const float* buf, const float* send_lo, float* recv_lo, const float* send_hi,
                    float* recv_hi, size_t n);
  void wait_halo(const float* buf);  // plan stream waits for buf's pending exchange
  void drain_halos();                // ... for every pending exchange
  void copy_image_x(float* dst, const float* src, size_t b);
  void fill_x_real(float* buf, size_t b, float v);
  int y_planes_total() const { return merged_ ? ny_user_planes_ : mz_ + 2 * pz_; }  // per image
  size_t xrun_elems() const {  // dense caller elements of one x run
    return xruns_.empty() ? 0 : static_cast<size_t>(xruns_[0].second) * my_ * mx_;
  }
  void copy_image_y(float* dst, const float* src, size_t b);
  void sync();
  void upload_active(const std::vector<int>& act);
  void upload_steps(const std::vector<double>& steps);
  void h2d_f64_as_f32(float* dev, const double* host, size_t n);
  void pack_dense_f64(const double* host, float* dev, const Vol& v, int z_off, int nz);
  void pack_dense_f32(const float* host, float* dev, const Vol& v, int z_off, int nz);
  void unpack_dense_f64(const float* dev, double* host, const Vol& v, int z_off, int nz);
  void unpack_dense_f32(const float* dev, float* host, const Vol& v, int z_off, int nz);
  float* x_owned(float* buf) const {
    return buf + X_.origin + static_cast<long long>(xa_ - xlo_) * X_.plane;
  }

  int device_ = 0;
  cudaStream_t stream_ = nullptr;
  size_t B_ = 1;
  int ndim_ = 1;
  size_t xext_[3] = {1, 1, 1}, kext_[3] = {1, 1, 1};  // the 3-d problem the kernels run
  std::vector<size_t> uext_x_, uext_k_;              // the caller's extents (any ndim)
  // ndim > 3: leading dims merged into the plane axis (see the constructor); x's real
  // planes are the runs xruns_ = (first owned plane, count), the rest stay zero
  bool merged_ = false;
  std::vector<std::pair<int, int>> xruns_;
  int ny_user_planes_ = 0;  // observation planes the caller passes (owned)
  double nreal_x_ = 0;      // x voxels per image (the caller's)
  int mz_ = 1, my_ = 1, mx_ = 1;
  int KZ_ = 1, KY_ = 1, KX_ = 1, pz_ = 0, py_ = 0, px_ = 0;
  int kcx_ = 1, kcy_ = 1;  // tap-chunk extents of one launch (x <= kMaxKX, rows <= TMA box)
  int ry_ = 1;      // output rows per thread in the correlation kernel (tile height 64*ry)
  int stages_ = 1;  // TMA plane stages in flight per CTA
  std::vector<float> taps_fwd_, taps_adj_;
  std::vector<double> h64_;     // the kernel as given (f64, flat)
  void set_taps(double scale);  // taps = float(h * scale), forward flipped, rows padded
  std::vector<TapChunk> build_chunks(const std::vector<float>& taps) const;
  std::vector<TapChunk> chunks_fwd_, chunks_adj_;
  bool kernel_all_zero_ = false;

  // z-slab geometry (global plane indices); unsharded: one slab holding everything.
  std::unique_ptr<Transport> comm_;
  int rank_ = 0, world_ = 1;
  int xa_ = 0, xb_ = 0, xa_n_ = 0;  // owned x planes
  int ya_ = 0, yb_ = 0;             // owned y planes
  int xlo_ = 0, xhi_ = 0;           // x planes held (owned + halo)
  int rlo_ = 0, rhi_ = 0;           // y planes held
  Vol X_, Y_;
  // halo exchanges run on their own stream, overlapped with the planes that need no halo
  cudaStream_t comm_stream_ = nullptr;
  // partial edge tiles of a pass run on a side stream (fork / join per pass)
  cudaStream_t edge_stream_ = nullptr;
  cudaEvent_t fork_ev_ = nullptr, join_ev_ = nullptr;
  cudaEvent_t pass_ev_ = nullptr;
  bool halo_overlap_ = true;
  std::map<const float*, cudaEvent_t> halo_ev_;
  std::set<const float*> halo_pending_;

  // device buffers
  float *x_ = nullptr, *trial_ = nullptr, *g_ = nullptr;
  float *trial2_ = nullptr, *g2_ = nullptr;  // speculative next-step adjoint outputs
  bool spec_ready_ = false;                  // this step's adjoint already ran speculatively
  cudaEvent_t d2h_ev_ = nullptr;
  float *yobs_ = nullptr, *r_ = nullptr, *rt_ = nullptr, *scratch_ = nullptr;
  double2* partials_ = nullptr;
  long long partials_cap_ = 0;
  double* dsc_ = nullptr;   // device scalars
  float* dscale_ = nullptr; // per-image scale
  int* dactive_ = nullptr;
  double* dstep_ = nullptr;
  double* gather_ = nullptr;
  double* hsc_ = nullptr;   // pinned host mirror of the device scalars
  double* hstep_ = nullptr;  // pinned upload mirrors (same block)
  int* hact_ = nullptr;
  size_t small_bytes_ = 0;
  cudaEvent_t up_ev_ = nullptr;
  size_t estimate_pending_ = 0;  // power_iters of a launched, uncollected estimate
  bool estimate_f64_ = false;
  double estimate_value_ = 0.0;
  std::vector<int> act_cache_;        // last uploaded per-image flags / steps
  std::vector<double> step_cache_;
  void* staging_ = nullptr;
  size_t staging_bytes_ = 0;
  std::map<std::pair<const float*, int>, CUtensorMap> maps_;

  // stats
  bool timing_ = false;
  KernelStats st_[3];
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pool_;
  std::vector<std::pair<int, size_t>> ev_pending_;  // (kind, pool index)
  size_t ev_used_ = 0;
  void drain_events();

  // PG state
  struct Img {
    std::vector<double> obj, kkt;
    double f = 0, step = 0;
    size_t iters = 0, backtracks = 0;
    int reason = NDC_STOP_MAX_ITERS;
    bool active = true;
    size_t clamped = 0;
  };
  std::vector<Img> img_;
  ndc_deconv_config cfg_{};
  double step0_ = 0;
  double wall0_ = 0, wall_ = 0;
  bool pg_begun_ = false;
};

}  // namespace ndc

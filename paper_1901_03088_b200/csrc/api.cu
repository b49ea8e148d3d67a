// api.cu — extern "C" entry points of libspcn.so (see include/spcn.h).
//
// Host-side validation mirrors the reference's argument checks so error
// behaviour is the same: validate_basis (src/stain_sep.py:89-101),
// beer_lambert's i0 check (src/optics.py:90-91), code_densities' lam check
// (src/stain_sep.py:188-189), normalize_block's factor check
// (src/normalize.py:141-142).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <condition_variable>
#include <mutex>
#include <utility>
#include <vector>
#include <string>

#include "spcn.h"
#include "spcn_device.cuh"
#include "params.cuh"
#include "xform.h"

#include "launch_count.h"

namespace spcn {
std::atomic<unsigned long long> g_launches{0};
}

using namespace spcn;

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* where) {
  return fail(SPCN_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

// validate_basis, src/stain_sep.py:89-101 (norm as np.linalg.norm: sqrt of the sum of squares)
int check_basis(const double* w, const char* role) {
  for (int k = 0; k < 6; ++k) {
    if (!std::isfinite(w[k])) return fail(SPCN_EINVAL, std::string(role) + " basis contains non-finite entries");
    if (w[k] < 0) return fail(SPCN_EINVAL, std::string(role) + " basis entries must be non-negative");
  }
  for (int j = 0; j < 2; ++j) {
    const double nrm = std::sqrt(w[0 * 2 + j] * w[0 * 2 + j] + w[1 * 2 + j] * w[1 * 2 + j] +
                                 w[2 * 2 + j] * w[2 * 2 + j]);
    if (std::fabs(nrm - 1.0) > 1e-9)
      return fail(SPCN_EINVAL, std::string(role) + " basis columns must have unit L2 norm");
  }
  return SPCN_OK;
}

// OD table: ln(i0_c / clip(i, 1, i0_c)), src/optics.py:92-94.
void od_table(const double* i0, const double* given, double lut[3][256]) {
  if (given) {
    std::memcpy(lut, given, sizeof(double) * 3 * 256);
    return;
  }
  for (int c = 0; c < 3; ++c)
    for (int i = 0; i < 256; ++i) {
      double x = static_cast<double>(i);
      x = x < 1.0 ? 1.0 : (x > i0[c] ? i0[c] : x);
      lut[c][i] = std::log(i0[c] / x);
    }
}

void fill_strict(StrictP& sp, const double* lut_src, const double* ws, const double* wt,
                 const double* f, const double* i0t, double lam, int max_sweeps) {
  std::memcpy(sp.lut, lut_src, sizeof(sp.lut));
  fill_strict_scalars(sp, ws, wt, f, i0t, lam, max_sweeps);
}

// fp32 coefficients + certification bound (params.cuh, shared with the batch builder)
bool fill_fast(FastP& fp, const StrictP& sp, bool exact) {
  return fill_fast_scalars(fp, sp, exact, fp.lut);
}

constexpr size_t kWsHeader = 16;

// Opt-in per-launch timing of the main recolor kernel (spcn_xform_timing_*).
std::atomic<int> g_timing{0};
std::mutex g_timing_mu;
std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_timing_ev;

void timing_begin(cudaStream_t st, cudaEvent_t& t0, cudaEvent_t& t1) {
  if (cudaEventCreate(&t0) != cudaSuccess || cudaEventCreate(&t1) != cudaSuccess) {
    t0 = t1 = nullptr;
    return;
  }
  cudaEventRecord(t0, st);
}

void timing_end(cudaStream_t st, cudaEvent_t t0, cudaEvent_t t1) {
  cudaEventRecord(t1, st);
  std::lock_guard<std::mutex> lk(g_timing_mu);
  g_timing_ev.emplace_back(t0, t1);
}

}  // namespace

extern "C" {

const char* spcn_last_error(void) { return g_err.c_str(); }

const char* spcn_version(void) { return "spcn-b200 0.1.0 (sm_100a)"; }

uint64_t spcn_launch_count(void) { return spcn::g_launches.load(std::memory_order_relaxed); }

const char* spcn_xform_shape(void) { return spcn::xform_shape_name(); }

int spcn_xform_timing_enable(int32_t on) {
  g_timing.store(on ? 1 : 0);
  return SPCN_OK;
}

int spcn_xform_timing(int64_t* launches, double* total_ms) {
  g_err.clear();
  if (!launches || !total_ms) return fail(SPCN_EINVAL, "NULL argument");
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev;
  {
    std::lock_guard<std::mutex> lk(g_timing_mu);
    ev.swap(g_timing_ev);
  }
  double sum = 0.0;
  cudaError_t err = cudaSuccess;
  for (auto& p : ev) {
    float ms = 0.f;
    cudaError_t e = cudaEventSynchronize(p.second);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, p.first, p.second);
    if (e != cudaSuccess && err == cudaSuccess) err = e;
    sum += ms;
    cudaEventDestroy(p.first);
    cudaEventDestroy(p.second);
  }
  *launches = static_cast<int64_t>(ev.size());
  *total_ms = sum;
  return err == cudaSuccess ? SPCN_OK : cuda_fail(err, "xform_timing");
}

size_t spcn_xform_workspace_bytes(int64_t npix) {
  const int64_t cap = 65536 + (npix > 0 ? npix / 32 : 0);
  return kWsHeader + static_cast<size_t>(cap) * 8;
}

}  // extern "C"

namespace {
// Validation shared by the transform entry points (see the file header).
int check_xform_params(const spcn_xform_params* p) {
  if (!p) return fail(SPCN_EINVAL, "params is NULL");
  if (p->precision < 0 || p->precision > 2) return fail(SPCN_EINVAL, "unknown precision");
  for (int c = 0; c < 3; ++c) {
    if (!(p->src_i0[c] >= 1.0) || !std::isfinite(p->src_i0[c]))
      return fail(SPCN_EINVAL, "i0 components must be >= 1");
    if (!std::isfinite(p->tgt_i0[c])) return fail(SPCN_EINVAL, "target i0 must be finite");
  }
  int rc = check_basis(p->src_basis, "source");
  if (rc) return rc;
  if ((rc = check_basis(p->tgt_basis, "target"))) return rc;
  if (!(p->code_lam >= 0.0)) return fail(SPCN_EINVAL, "lam must be >= 0");
  for (int j = 0; j < 2; ++j)
    if (!(p->factors[j] > 0.0) || !std::isfinite(p->factors[j]))
      return fail(SPCN_EINVAL, "factors must be positive and finite");
  if (p->max_sweeps < 0) return fail(SPCN_EINVAL, "max_sweeps must be >= 0");
  return SPCN_OK;
}

// Calibrated certification interval bounds (rounded outward in fp32).
void set_calibrated(FastP& fp, double alpha) {
  fp.a1 = 0.0f;
  fp.a0 = static_cast<float>(alpha);
  for (int c = 0; c < 3; ++c) {
    const double i0 = static_cast<double>(fp.i0t[c]);
    float lo = static_cast<float>(i0 * (1.0 - alpha));
    float hi = static_cast<float>(i0 * (1.0 + alpha));
    lo = std::nextafter(lo, 0.0f);
    hi = std::nextafter(hi, 1e30f);
    fp.I[c].x = lo;
    fp.I[c].y = hi;
  }
}
}  // namespace

extern "C" {

int spcn_xform_calibrate(const spcn_xform_params* p, void* workspace, size_t workspace_bytes,
                         double* alpha_out, void* stream) {
  g_err.clear();
  int rc = check_xform_params(p);
  if (rc) return rc;
  if (!alpha_out) return fail(SPCN_EINVAL, "alpha_out is NULL");
  if (!workspace || workspace_bytes < kWsHeader) return fail(SPCN_EINVAL, "workspace too small");
  double lut[3][256];
  od_table(p->src_i0, p->od_table, lut);
  static thread_local StrictP sp;
  static thread_local FastP fp;
  fill_strict(sp, &lut[0][0], p->src_basis, p->tgt_basis, p->factors, p->tgt_i0, p->code_lam,
              p->max_sweeps);
  *alpha_out = -1.0;
  if (!fill_fast(fp, sp, true)) return SPCN_OK;   // fast path not applicable: strict is used
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned int* bits = static_cast<unsigned int*>(workspace);
  cudaError_t e = cudaMemsetAsync(bits, 0, sizeof(unsigned int), st);
  if (e == cudaSuccess) e = launch_calibrate(fp, sp, bits, st);
  unsigned int h = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&h, bits, sizeof(h), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_fail(e, "xform_calibrate");
  float worst;
  std::memcpy(&worst, &h, sizeof(worst));
  // The exhaustive sweep ran the transform's own fast path on every colour, so
  // the worst observed relative error IS the bound; the factor only absorbs
  // the fp32 rounding of `worst` (set_calibrated rounds the interval ends
  // outward).  DESIGN.md §Certified rounding.
  const double alpha = static_cast<double>(worst) * (1.0 + std::ldexp(1.0, -20));
  // a calibrated bound looser than the analytic one is never used
  *alpha_out = alpha < 1e-3 ? alpha : -1.0;
  return SPCN_OK;
}

int spcn_xform_rgb8(const uint8_t* src, uint8_t* dst, int64_t npix, const spcn_xform_params* p,
                    void* workspace, size_t workspace_bytes, void* stream) {
  g_err.clear();
  if (!p) return fail(SPCN_EINVAL, "params is NULL");
  if (npix < 0) return fail(SPCN_EINVAL, "npix must be >= 0");
  if (npix == 0) return SPCN_OK;
  if (!src || !dst) return fail(SPCN_EINVAL, "src/dst is NULL");
  if (p->precision < 0 || p->precision > 2) return fail(SPCN_EINVAL, "unknown precision");
  for (int c = 0; c < 3; ++c) {
    if (!(p->src_i0[c] >= 1.0) || !std::isfinite(p->src_i0[c]))
      return fail(SPCN_EINVAL, "i0 components must be >= 1");
    if (!std::isfinite(p->tgt_i0[c])) return fail(SPCN_EINVAL, "target i0 must be finite");
  }
  int rc = check_basis(p->src_basis, "source");
  if (rc) return rc;
  if ((rc = check_basis(p->tgt_basis, "target"))) return rc;
  if (!(p->code_lam >= 0.0)) return fail(SPCN_EINVAL, "lam must be >= 0");
  for (int j = 0; j < 2; ++j)
    if (!(p->factors[j] > 0.0) || !std::isfinite(p->factors[j]))
      return fail(SPCN_EINVAL, "factors must be positive and finite");
  if (p->max_sweeps < 0) return fail(SPCN_EINVAL, "max_sweeps must be >= 0");

  double lut[3][256];
  od_table(p->src_i0, p->od_table, lut);
  static thread_local StrictP sp;
  static thread_local FastP fp;
  fill_strict(sp, &lut[0][0], p->src_basis, p->tgt_basis, p->factors, p->tgt_i0, p->code_lam,
              p->max_sweeps);
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool exact = p->precision == SPCN_PREC_EXACT;
  bool fast_ok = p->precision != SPCN_PREC_STRICT && fill_fast(fp, sp, exact);
  int mode = exact ? 0 : 1;
  // cert_alpha == SPCN_CALIBRATE_INLINE: calibrate on the device right before
  // the main kernel, which reads the result itself (no host round trip)
  const bool inline_cal = exact && fast_ok && p->cert_alpha == SPCN_CALIBRATE_INLINE;
  // SPCN_CALIBRATE_DEVICE: the calibration word is already in the workspace
  // (spcn_xform_calibrate_part on every rank + an all-reduce max)
  const bool device_cal = exact && fast_ok && p->cert_alpha == SPCN_CALIBRATE_DEVICE;
  if (exact && fast_ok && p->cert_alpha > 0.0 && p->cert_alpha < 1e-3) {
    set_calibrated(fp, p->cert_alpha);
    mode = 2;
  }
  if (inline_cal || device_cal) mode = 2;

  // 16-byte alignment of the vector body (both buffers must share the phase)
  const uintptr_t sa = reinterpret_cast<uintptr_t>(src), da = reinterpret_cast<uintptr_t>(dst);
  if (((sa - da) & 15u) != 0) fast_ok = false;
  int64_t head = static_cast<int64_t>(((16 - (sa & 15u)) * 11u) & 15u);  // 3*head == -sa (mod 16)
  if (head > npix) head = npix;
  const int64_t body = fast_ok ? ((npix - head) / 16) * 16 : 0;
  if (!fast_ok || body == 0) {
    cudaError_t e = launch_xform_strict(src, dst, npix, sp, st);
    return e == cudaSuccess ? SPCN_OK : cuda_fail(e, "xform_strict");
  }
  unsigned long long* count = nullptr;
  unsigned long long* items = nullptr;
  unsigned long long cap = 0;
  if (exact) {
    if (!workspace || workspace_bytes < kWsHeader + 8)
      return fail(SPCN_EINVAL, "EXACT precision needs a workspace (spcn_xform_workspace_bytes)");
    count = static_cast<unsigned long long*>(workspace);
    items = reinterpret_cast<unsigned long long*>(static_cast<char*>(workspace) + kWsHeader);
    cap = (workspace_bytes - kWsHeader) / 8;
    // count + calibration word (kept when it was computed beforehand)
    cudaError_t e = cudaMemsetAsync(count, 0, device_cal ? 8 : kWsHeader, st);
    if (e != cudaSuccess) return cuda_fail(e, "memset");
  }
  cudaError_t e;
  const unsigned int* alpha_bits = nullptr;
  if (inline_cal) {
    unsigned int* bits = reinterpret_cast<unsigned int*>(static_cast<char*>(workspace) + 8);
    if ((e = launch_calibrate(fp, sp, bits, st)) != cudaSuccess) return cuda_fail(e, "calibrate");
    alpha_bits = bits;
  }
  if (device_cal)
    alpha_bits = reinterpret_cast<const unsigned int*>(static_cast<char*>(workspace) + 8);
  if (head > 0 && (e = launch_xform_strict(src, dst, head, sp, st)) != cudaSuccess)
    return cuda_fail(e, "xform_head");
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  if (g_timing.load(std::memory_order_relaxed)) timing_begin(st, t0, t1);
  e = launch_xform_main(mode, src + 3 * head, dst + 3 * head, body, fp, sp, count, items, cap,
                        alpha_bits, st);
  if (t0) timing_end(st, t0, t1);
  if (e != cudaSuccess) return cuda_fail(e, "xform_tma");
  if (exact && (e = launch_xform_repair(src + 3 * head, dst + 3 * head, body, sp, count, items, cap,
                                        st)) != cudaSuccess)
    return cuda_fail(e, "xform_repair");
  const int64_t tail0 = head + body;
  if (tail0 < npix &&
      (e = launch_xform_strict(src + 3 * tail0, dst + 3 * tail0, npix - tail0, sp, st)) != cudaSuccess)
    return cuda_fail(e, "xform_tail");
  return SPCN_OK;
}

int spcn_xform_calibrate_part(const spcn_xform_params* p, int32_t part, int32_t nparts,
                              void* workspace, int64_t workspace_bytes, void* stream) {
  g_err.clear();
  if (!p) return fail(SPCN_EINVAL, "params is NULL");
  if (nparts < 1 || part < 0 || part >= nparts) return fail(SPCN_EINVAL, "bad part");
  if (!workspace || workspace_bytes < kWsHeader) return fail(SPCN_EINVAL, "workspace too small");
  int rc = check_basis(p->src_basis, "source");
  if (!rc) rc = check_basis(p->tgt_basis, "target");
  if (rc) return rc;
  double lut[3][256];
  od_table(p->src_i0, p->od_table, lut);
  static thread_local StrictP sp;
  static thread_local FastP fp;
  fill_strict(sp, &lut[0][0], p->src_basis, p->tgt_basis, p->factors, p->tgt_i0, p->code_lam,
              p->max_sweeps);
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  unsigned int* bits = reinterpret_cast<unsigned int*>(static_cast<char*>(workspace) + 8);
  cudaError_t e = cudaMemsetAsync(bits, 0, 4, st);
  if (e != cudaSuccess) return cuda_fail(e, "memset");
  if (!fill_fast(fp, sp, true)) return SPCN_OK;   // no fast path: the word stays 0 (unused)
  const uint32_t n = 1u << 23;
  const uint32_t q0 = static_cast<uint32_t>((uint64_t)n * part / nparts),
                 q1 = static_cast<uint32_t>((uint64_t)n * (part + 1) / nparts);
  e = launch_calibrate(fp, sp, bits, st, q0, q1);
  return e == cudaSuccess ? SPCN_OK : cuda_fail(e, "calibrate_part");
}

}  // extern "C"

namespace {
// Parameter slots of the device-built recolouring, per device: slot k's
// staging block and __constant__ copy may be rewritten only after the
// previous recolouring that used slot k has finished (its event).
struct FittedSlots {
  DevParams* staging = nullptr;           // kDpSlots blocks
  cudaEvent_t done[kDpSlots] = {};
  cudaEvent_t built[kDpSlots] = {};       // the status read-back has landed
  bool used[kDpSlots] = {};
  bool analytic[kDpSlots] = {};           // the slot's recolouring uses the analytic bound
  // prepared, its run not yet enqueued: `done` does not cover the slot's
  // recolour yet, so another prepare must not take the slot (threads that
  // prepare concurrently block here until the run is enqueued)
  bool pending[kDpSlots] = {};
  int next = 0;
};
std::mutex g_fitted_mu;
std::condition_variable g_fitted_cv;
FittedSlots g_fitted[64];

int check_fitted(const spcn_xform_fitted* p) {
  if (!p) return fail(SPCN_EINVAL, "params is NULL");
  if (!p->src_od_table || !p->src_fit) return fail(SPCN_EINVAL, "NULL table / fit arena");
  if (p->tgt_fit && !p->tgt_i0_dev) return fail(SPCN_EINVAL, "tgt_fit needs tgt_i0_dev");
  if (!p->tgt_fit) {   // a host-side target profile (a device-side one is checked on the device)
    int rc = check_basis(p->tgt_basis, "target");
    if (rc) return rc;
    for (int c = 0; c < 3; ++c)
      if (!std::isfinite(p->tgt_i0[c])) return fail(SPCN_EINVAL, "target i0 must be finite");
    for (int j = 0; j < 2; ++j)
      if (!(p->tgt_p99[j] > 0.0) || !std::isfinite(p->tgt_p99[j]))
        return fail(SPCN_EINVAL, "target p99 must be positive and finite");
  }
  if (!(p->code_lam >= 0.0)) return fail(SPCN_EINVAL, "lam must be >= 0");
  if (p->max_sweeps < 0) return fail(SPCN_EINVAL, "max_sweeps must be >= 0");
  if (p->flags & ~SPCN_FITTED_ANALYTIC) return fail(SPCN_EINVAL, "unknown flags");
  return SPCN_OK;
}

void release_slot(int dev, int slot) {
  {
    std::lock_guard<std::mutex> lk(g_fitted_mu);
    g_fitted[dev].pending[slot] = false;
  }
  g_fitted_cv.notify_all();
}

// slot + build + calibration part; *built_out = the event after the status read-back
int fitted_prepare(const spcn_xform_fitted* p, int32_t part, int32_t nparts, void* workspace,
                   size_t workspace_bytes, int32_t* status_pinned, cudaStream_t st,
                   int32_t* slot_out, cudaEvent_t* built_out) {
  int rc = check_fitted(p);
  if (rc) return rc;
  if (nparts < 1 || part < 0 || part >= nparts) return fail(SPCN_EINVAL, "bad part");
  if (!workspace || workspace_bytes < kWsHeader + 8)
    return fail(SPCN_EINVAL, "workspace too small (spcn_xform_workspace_bytes)");
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "get_device");
  if (dev < 0 || dev >= 64) return fail(SPCN_EINVAL, "device index out of range");
  int slot;
  DevParams* staging;
  cudaEvent_t built;
  {
    std::unique_lock<std::mutex> lk(g_fitted_mu);
    FittedSlots& fs = g_fitted[dev];
    if (!fs.staging) {
      if ((e = cudaMalloc(&fs.staging, sizeof(DevParams) * kDpSlots)) != cudaSuccess)
        return cuda_fail(e, "staging alloc");
      for (int k = 0; k < kDpSlots; ++k)
        if ((e = cudaEventCreateWithFlags(&fs.done[k], cudaEventDisableTiming)) != cudaSuccess ||
            (e = cudaEventCreateWithFlags(&fs.built[k], cudaEventDisableTiming)) != cudaSuccess)
          return cuda_fail(e, "event");
    }
    g_fitted_cv.wait(lk, [&] {   // the next slot in ring order that is not pending
      for (int k = 0; k < kDpSlots; ++k)
        if (!fs.pending[(fs.next + k) % kDpSlots]) return true;
      return false;
    });
    slot = fs.next;
    while (fs.pending[slot]) slot = (slot + 1) % kDpSlots;
    fs.next = (slot + 1) % kDpSlots;
    staging = fs.staging + slot;
    built = fs.built[slot];
    // the slot's previous user (any stream) must be finished with it
    if (fs.used[slot] && (e = cudaStreamWaitEvent(st, fs.done[slot], 0)) != cudaSuccess)
      return cuda_fail(e, "slot wait");
    fs.used[slot] = true;
    fs.pending[slot] = true;
    fs.analytic[slot] = (p->flags & SPCN_FITTED_ANALYTIC) != 0;
  }
  XformBuildIn in{};
  std::memcpy(in.tgt_basis, p->tgt_basis, sizeof(in.tgt_basis));
  std::memcpy(in.tgt_p99, p->tgt_p99, sizeof(in.tgt_p99));
  std::memcpy(in.tgt_i0, p->tgt_i0, sizeof(in.tgt_i0));
  in.code_lam = p->code_lam;
  in.max_sweeps = p->max_sweeps;
  in.tgt_fit_dev = static_cast<const double*>(p->tgt_fit);
  in.tgt_i0_dev = p->tgt_fit ? p->tgt_i0_dev : nullptr;
  const uint32_t n = (p->flags & SPCN_FITTED_ANALYTIC) ? 0u : 1u << 23;   // colour pairs
  const uint32_t q0 = static_cast<uint32_t>((uint64_t)n * part / nparts),
                 q1 = static_cast<uint32_t>((uint64_t)n * (part + 1) / nparts);
  if ((e = launch_xform_build(slot, in, p->src_od_table, static_cast<const double*>(p->src_fit),
                              staging, workspace, status_pinned, built, q0, q1, st)) != cudaSuccess) {
    release_slot(dev, slot);
    return cuda_fail(e, "xform_build");
  }
  *slot_out = slot;
  *built_out = built;
  return SPCN_OK;
}

int fitted_run_launch(const uint8_t* src, uint8_t* dst, int64_t npix, int32_t slot, bool analytic,
                      void* workspace, size_t workspace_bytes, cudaStream_t st) {
  cudaError_t e;
  if (npix > 0) {
    if (!src || !dst) return fail(SPCN_EINVAL, "src/dst is NULL");
    const uintptr_t sa = reinterpret_cast<uintptr_t>(src), da = reinterpret_cast<uintptr_t>(dst);
    if (((sa - da) & 15u) != 0)
      return fail(SPCN_EINVAL, "src and dst must share their 16-byte alignment phase");
    if (!workspace || workspace_bytes < spcn_xform_workspace_bytes(npix))
      return fail(SPCN_EINVAL, "workspace too small (spcn_xform_workspace_bytes)");
    char* ws = static_cast<char*>(workspace);
    int64_t head = static_cast<int64_t>(((16 - (sa & 15u)) * 11u) & 15u);   // 3*head == -sa (mod 16)
    if (head > npix) head = npix;
    const int64_t body = ((npix - head) / 16) * 16;
    auto* count = reinterpret_cast<unsigned long long*>(ws);
    auto* items = reinterpret_cast<unsigned long long*>(ws + kWsHeader);
    const unsigned long long cap = (workspace_bytes - kWsHeader) / 8;
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    if (g_timing.load(std::memory_order_relaxed)) timing_begin(st, t0, t1);
    e = launch_xform_main_c(slot, analytic, src + 3 * head, dst + 3 * head, body, count, items,
                            cap, reinterpret_cast<const unsigned int*>(ws + 8), st);
    if (t0) timing_end(st, t0, t1);
    if (e != cudaSuccess) return cuda_fail(e, "xform_main_c");
    if ((e = launch_xform_repair_c(slot, src, dst, npix, head, body, count, items, cap, st)) !=
        cudaSuccess)
      return cuda_fail(e, "xform_repair_c");
  }
  return SPCN_OK;
}

// The recolour of a prepared slot; on every path the slot's `done` event is
// recorded (covering its build and recolour) and the slot released.
int fitted_run(const uint8_t* src, uint8_t* dst, int64_t npix, int32_t slot, void* workspace,
               size_t workspace_bytes, cudaStream_t st) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_fail(e, "get_device");
  if (dev < 0 || dev >= 64) return fail(SPCN_EINVAL, "device index out of range");
  if (slot < 0 || slot >= kDpSlots) return fail(SPCN_EINVAL, "bad slot");
  cudaEvent_t done;
  bool analytic;
  {
    std::lock_guard<std::mutex> lk(g_fitted_mu);
    if (!g_fitted[dev].staging) return fail(SPCN_EINVAL, "no prepared recolouring");
    done = g_fitted[dev].done[slot];
    analytic = g_fitted[dev].analytic[slot];
  }
  const int rc = fitted_run_launch(src, dst, npix, slot, analytic, workspace, workspace_bytes, st);
  e = cudaEventRecord(done, st);
  release_slot(dev, slot);
  if (rc) return rc;
  if (e != cudaSuccess) return cuda_fail(e, "slot record");
  return SPCN_OK;
}

}  // namespace

extern "C" {

int spcn_xform_fitted_prepare(const spcn_xform_fitted* p, int32_t part, int32_t nparts,
                              void* workspace, size_t workspace_bytes, int32_t* status_pinned,
                              int32_t* slot_out, void* stream) {
  g_err.clear();
  if (!slot_out) return fail(SPCN_EINVAL, "slot_out is NULL");
  cudaEvent_t built = nullptr;
  int rc = fitted_prepare(p, part, nparts, workspace, workspace_bytes, status_pinned,
                          static_cast<cudaStream_t>(stream), slot_out, &built);
  if (rc) return rc;
  cudaError_t e;
  if (status_pinned && (e = cudaEventSynchronize(built)) != cudaSuccess)
    return cuda_fail(e, "build wait");
  return SPCN_OK;
}

int spcn_xform_fitted_run(const uint8_t* src, uint8_t* dst, int64_t npix, int32_t slot,
                          void* workspace, size_t workspace_bytes, void* stream) {
  g_err.clear();
  if (npix < 0) return fail(SPCN_EINVAL, "npix must be >= 0");
  return fitted_run(src, dst, npix, slot, workspace, workspace_bytes,
                    static_cast<cudaStream_t>(stream));
}

int spcn_xform_rgb8_fitted(const uint8_t* src, uint8_t* dst, int64_t npix,
                           const spcn_xform_fitted* p, void* workspace, size_t workspace_bytes,
                           int32_t* status_pinned, void* stream) {
  g_err.clear();
  if (npix <= 0) return fail(SPCN_EINVAL, "npix must be > 0");
  if (!src || !dst) return fail(SPCN_EINVAL, "src/dst is NULL");
  const uintptr_t sa = reinterpret_cast<uintptr_t>(src), da = reinterpret_cast<uintptr_t>(dst);
  if (((sa - da) & 15u) != 0)
    return fail(SPCN_EINVAL, "src and dst must share their 16-byte alignment phase");
  if (!workspace || workspace_bytes < spcn_xform_workspace_bytes(npix))
    return fail(SPCN_EINVAL, "workspace too small (spcn_xform_workspace_bytes)");
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  int32_t slot = 0;
  cudaEvent_t built = nullptr;
  int rc = fitted_prepare(p, 0, 1, workspace, workspace_bytes, status_pinned, st, &slot, &built);
  if (rc) return rc;
  if ((rc = fitted_run(src, dst, npix, slot, workspace, workspace_bytes, st))) return rc;
  // the build (and everything enqueued before it, e.g. the fit's read-back)
  // has reached host memory; the recolour itself is still in flight
  cudaError_t e;
  if (status_pinned && (e = cudaEventSynchronize(built)) != cudaSuccess)
    return cuda_fail(e, "build wait");
  return SPCN_OK;
}

int spcn_xform_repair_count(const void* workspace, void* stream, int64_t* count) {
  g_err.clear();
  if (!workspace || !count) return fail(SPCN_EINVAL, "NULL argument");
  unsigned long long c = 0;
  cudaError_t e = cudaMemcpyAsync(&c, workspace, sizeof(c), cudaMemcpyDeviceToHost,
                                  static_cast<cudaStream_t>(stream));
  if (e == cudaSuccess) e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "repair_count");
  *count = static_cast<int64_t>(c);
  return SPCN_OK;
}

int spcn_code_densities(const double* od, double* h, int64_t n, const double* basis, double lam,
                        int32_t max_sweeps, void* stream) {
  g_err.clear();
  if (n < 0) return fail(SPCN_EINVAL, "n must be >= 0");
  if (!basis) return fail(SPCN_EINVAL, "basis is NULL");
  int rc = check_basis(basis, "stain");
  if (rc) return rc;
  if (!(lam >= 0.0)) return fail(SPCN_EINVAL, "lam must be >= 0");
  if (max_sweeps < 0) return fail(SPCN_EINVAL, "max_sweeps must be >= 0");
  if (n == 0) return SPCN_OK;
  if (!od || !h) return fail(SPCN_EINVAL, "od/h is NULL");
  static thread_local StrictP sp;
  static const double zero_lut[3 * 256] = {0};
  fill_strict(sp, zero_lut, basis, nullptr, nullptr, nullptr, lam, max_sweeps);
  cudaError_t e = launch_code_densities(od, h, n, sp, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SPCN_OK : cuda_fail(e, "code_densities");
}

int spcn_normalize_block(const double* h, uint8_t* out, int64_t n, const double* factors,
                         const double* tgt_basis, const double* tgt_i0, void* stream) {
  g_err.clear();
  if (n < 0) return fail(SPCN_EINVAL, "n must be >= 0");
  if (!factors || !tgt_basis || !tgt_i0) return fail(SPCN_EINVAL, "NULL argument");
  int rc = check_basis(tgt_basis, "target");
  if (rc) return rc;
  for (int j = 0; j < 2; ++j)
    if (!(factors[j] > 0.0) || !std::isfinite(factors[j]))
      return fail(SPCN_EINVAL, "factors must be positive and finite");
  if (n == 0) return SPCN_OK;
  if (!h || !out) return fail(SPCN_EINVAL, "h/out is NULL");
  static thread_local StrictP sp;
  static const double zero_lut[3 * 256] = {0};
  fill_strict(sp, zero_lut, nullptr, tgt_basis, factors, tgt_i0, 0.0, 0);
  cudaError_t e = launch_normalize_block(h, out, n, sp, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SPCN_OK : cuda_fail(e, "normalize_block");
}

int spcn_beer_lambert(const uint8_t* px, double* od, int64_t n, const double* i0,
                      const double* od_table_in, void* stream) {
  g_err.clear();
  if (n < 0) return fail(SPCN_EINVAL, "n must be >= 0");
  if (!i0) return fail(SPCN_EINVAL, "i0 is NULL");
  for (int c = 0; c < 3; ++c)
    if (!(i0[c] >= 1.0)) return fail(SPCN_EINVAL, "i0 components must be >= 1");
  if (n == 0) return SPCN_OK;
  if (!px || !od) return fail(SPCN_EINVAL, "px/od is NULL");
  double lut[3][256];
  od_table(i0, od_table_in, lut);
  static thread_local StrictP sp;
  fill_strict(sp, &lut[0][0], nullptr, nullptr, nullptr, nullptr, 0.0, 0);
  cudaError_t e = launch_beer_lambert(px, od, n, sp, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SPCN_OK : cuda_fail(e, "beer_lambert");
}

int spcn_inverse_beer_lambert(const double* od, uint8_t* out, int64_t n, const double* i0,
                              void* stream) {
  g_err.clear();
  if (n < 0) return fail(SPCN_EINVAL, "n must be >= 0");
  if (!i0) return fail(SPCN_EINVAL, "i0 is NULL");
  if (n == 0) return SPCN_OK;
  if (!od || !out) return fail(SPCN_EINVAL, "od/out is NULL");
  static thread_local StrictP sp;
  static const double zero_lut[3 * 256] = {0};
  fill_strict(sp, zero_lut, nullptr, nullptr, nullptr, i0, 0.0, 0);
  cudaError_t e = launch_inverse_bl(od, out, n, sp, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SPCN_OK : cuda_fail(e, "inverse_beer_lambert");
}

}  // extern "C"

// ------------------------------------------------------------------ fit entry points
#include "sample.h"
#include "select.h"
#include "snmf.h"

extern "C" {

int spcn_sample_count(const uint8_t* img, const spcn_patch* patches, int32_t npatches,
                      int32_t max_chunks, int32_t white_threshold, int32_t* counts,
                      void* stream) {
  g_err.clear();
  if (npatches < 0 || max_chunks < 0) return fail(SPCN_EINVAL, "negative size");
  if (npatches == 0) return SPCN_OK;
  if (!img || !patches || !counts) return fail(SPCN_EINVAL, "NULL argument");
  cudaError_t e = launch_sample_count(img, patches, npatches, max_chunks, white_threshold, counts,
                                      static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SPCN_OK : cuda_fail(e, "sample_count");
}

int spcn_visit_single(const int32_t* counts, int32_t n, int32_t chunks, double used_min,
                      int64_t target, int64_t cap, spcn_patch_take* takes, int64_t* take_nw,
                      void* stream) {
  g_err.clear();
  if (n < 0 || chunks < 1) return fail(SPCN_EINVAL, "bad size");
  if (n == 0) return SPCN_OK;
  if (!counts || !takes || !take_nw) return fail(SPCN_EINVAL, "NULL argument");
  if (target < 0 || cap < 0) return fail(SPCN_EINVAL, "negative take");
  cudaError_t e = launch_visit_single(counts, n, chunks, used_min, target, cap, takes, take_nw,
                                      static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SPCN_OK : cuda_fail(e, "visit_single");
}

int spcn_sample_compact(const uint8_t* img, const spcn_patch* patches, int32_t npatches,
                        int32_t max_chunks, int32_t white_threshold, const int32_t* counts,
                        const spcn_patch_take* takes, uint8_t* out_px, int32_t* bright_hist,
                        void* stream) {
  g_err.clear();
  if (npatches < 0 || max_chunks < 0) return fail(SPCN_EINVAL, "negative size");
  if (npatches == 0) return SPCN_OK;
  if (!img || !patches || !counts || !takes || !bright_hist) return fail(SPCN_EINVAL, "NULL argument");
  cudaError_t e = launch_sample_compact(img, patches, npatches, max_chunks, white_threshold, counts,
                                        takes, out_px, bright_hist,
                                        static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SPCN_OK : cuda_fail(e, "sample_compact");
}

int spcn_sample_visit(const int32_t* counts, int32_t n, int32_t max_chunks, int32_t k0,
                      const int32_t* dims, const spcn_visit_plan* plan, int64_t* state,
                      spcn_patch_take* takes, int64_t* offsets, void* stream) {
  g_err.clear();
  if (n < 1 || n > 4096 || max_chunks < 1 || k0 < 0) return fail(SPCN_EINVAL, "bad batch");
  if (!counts || !dims || !plan || !state || !takes || !offsets)
    return fail(SPCN_EINVAL, "NULL argument");
  if (plan->max_patches < 1 || plan->target_pixels < 1 || plan->sample_cap < 0)
    return fail(SPCN_EINVAL, "bad sample plan");
  const cudaError_t e = launch_visit(counts, n, max_chunks, k0, dims, *plan, state, takes, offsets,
                                     static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SPCN_OK : cuda_fail(e, "sample_visit");
}

int spcn_i0_from_hist(const int32_t* hist, int32_t nprob, double* i0, int32_t* empty,
                      void* stream) {
  g_err.clear();
  if (nprob < 0) return fail(SPCN_EINVAL, "negative size");
  if (nprob == 0) return SPCN_OK;
  if (!hist || !i0 || !empty) return fail(SPCN_EINVAL, "NULL argument");
  cudaError_t e = launch_i0_from_hist(hist, nprob, i0, empty, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SPCN_OK : cuda_fail(e, "i0_from_hist");
}

int spcn_od_tables(const double* i0, int32_t nprob, double* lut, void* stream) {
  g_err.clear();
  if (nprob < 0) return fail(SPCN_EINVAL, "negative size");
  if (nprob == 0) return SPCN_OK;
  if (!i0 || !lut) return fail(SPCN_EINVAL, "NULL argument");
  cudaError_t e = launch_od_tables(i0, nprob, lut, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SPCN_OK : cuda_fail(e, "od_tables");
}

int spcn_snmf_batched(const uint8_t* samples, const double* od, const int64_t* offsets,
                      int32_t nprob,
                      const double* luts, const spcn_snmf_cfg* cfg, double* hscratch,
                      int64_t total, double* basis_out, double* history_out, int32_t* info_out,
                      void* stream) {
  g_err.clear();
  if (!cfg) return fail(SPCN_EINVAL, "cfg is NULL");
  if (nprob < 0 || total < 0) return fail(SPCN_EINVAL, "negative size");
  if (!(cfg->lam >= 0.0)) return fail(SPCN_EINVAL, "lam must be >= 0");
  if (cfg->max_outer < 1) return fail(SPCN_EINVAL, "max_outer_iters must be >= 1");
  if (!(cfg->rel_tol > 0.0)) return fail(SPCN_EINVAL, "rel_tol must be > 0");
  if (cfg->cluster < 1 || cfg->cluster > 16) return fail(SPCN_EINVAL, "cluster must be in [1, 16]");
  if (nprob == 0) return SPCN_OK;
  if ((!od && (!samples || !luts)) || !offsets || !basis_out || !history_out || !info_out)
    return fail(SPCN_EINVAL, "NULL argument");
  SnmfArgs a;
  a.lam = cfg->lam;
  a.rel_tol = cfg->rel_tol;
  for (int i = 0; i < 6; ++i) a.w_init[i] = cfg->w_init[i];
  a.max_outer = cfg->max_outer;
  a.pad_ = 0;
  cudaError_t e = launch_snmf(samples, od, offsets, nprob, luts, a, hscratch, total, basis_out,
                              history_out, info_out, cfg->cluster,
                              static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SPCN_OK : cuda_fail(e, "snmf");
}

int spcn_code_samples(const uint8_t* samples, const int64_t* offsets, int32_t nprob,
                      int64_t max_m, const double* luts, const double* bases, double lam,
                      int32_t max_sweeps, double* h, int64_t total, void* stream) {
  g_err.clear();
  if (nprob < 0 || total < 0) return fail(SPCN_EINVAL, "negative size");
  if (!(lam >= 0.0)) return fail(SPCN_EINVAL, "lam must be >= 0");
  if (max_sweeps < 0) return fail(SPCN_EINVAL, "max_sweeps must be >= 0");
  if (nprob == 0 || total == 0) return SPCN_OK;
  if (!samples || !offsets || !luts || !bases || !h) return fail(SPCN_EINVAL, "NULL argument");
  cudaError_t e = launch_code_samples(samples, offsets, nprob, max_m, luts, bases, lam, max_sweeps,
                                      h, total, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SPCN_OK : cuda_fail(e, "code_samples");
}

int spcn_code_table(const void* hscratch, const int64_t* offsets, int32_t nprob, int64_t max_m,
                    const double* luts, const double* bases, double lam, int32_t max_sweeps,
                    double* h, int64_t total, void* stream) {
  g_err.clear();
  if (nprob < 0 || total < 0) return fail(SPCN_EINVAL, "negative size");
  if (!(lam >= 0.0)) return fail(SPCN_EINVAL, "lam must be >= 0");
  if (max_sweeps < 0) return fail(SPCN_EINVAL, "max_sweeps must be >= 0");
  if (nprob == 0 || total == 0) return SPCN_OK;
  if (!hscratch || !offsets || !luts || !bases || !h) return fail(SPCN_EINVAL, "NULL argument");
  const uint32_t* ukey = static_cast<const uint32_t*>(hscratch);
  const int32_t* ucount = reinterpret_cast<const int32_t*>(ukey + 2 * total);
  cudaError_t e = launch_code_table(ukey, ucount, offsets, nprob, max_m, luts, bases, lam,
                                    max_sweeps, h, total, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SPCN_OK : cuda_fail(e, "code_table");
}

int spcn_percentile_table(const double* h, int64_t total, const void* hscratch,
                          const int64_t* seg_offsets, int32_t nseg, double p, double* out,
                          int32_t* absent, void* stream) {
  g_err.clear();
  if (nseg < 0 || total < 0) return fail(SPCN_EINVAL, "negative size");
  if (!(p >= 0.0 && p <= 100.0)) return fail(SPCN_EINVAL, "percentile p must be in [0, 100]");
  if (nseg == 0) return SPCN_OK;
  if (!h || !hscratch || !seg_offsets || !out || !absent) return fail(SPCN_EINVAL, "NULL argument");
  const uint32_t* ukey = static_cast<const uint32_t*>(hscratch);
  const uint32_t* ucnt = ukey + total;
  const int32_t* ucount = reinterpret_cast<const int32_t*>(ukey + 2 * total);
  cudaError_t e = launch_p99_weighted(h, total, ucnt, ucount, seg_offsets, nseg, p, out, absent,
                                      static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SPCN_OK : cuda_fail(e, "percentile_table");
}

int spcn_percentile_segments(const double* h, int64_t total, const int64_t* seg_offsets,
                             int32_t nseg, double p, void* qbuf, double* selbuf, double* out,
                             int32_t* absent, void* stream) {
  g_err.clear();
  if (nseg < 0 || total < 0) return fail(SPCN_EINVAL, "negative size");
  if (!(p >= 0.0 && p <= 100.0)) return fail(SPCN_EINVAL, "percentile p must be in [0, 100]");
  if (nseg == 0) return SPCN_OK;
  if (!h || !seg_offsets || !qbuf || !selbuf || !out || !absent)
    return fail(SPCN_EINVAL, "NULL argument");
  cudaError_t e = launch_p99(h, total, seg_offsets, nseg, p, static_cast<SelQuery*>(qbuf), selbuf,
                             out, absent, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SPCN_OK : cuda_fail(e, "percentile_segments");
}

int spcn_select_kth(const double* values, const int64_t* begin, const int64_t* end,
                    const int64_t* k, int32_t nq, void* qbuf, double* out, void* stream) {
  g_err.clear();
  if (nq < 0) return fail(SPCN_EINVAL, "negative size");
  if (nq == 0) return SPCN_OK;
  if (!values || !begin || !end || !k || !qbuf || !out) return fail(SPCN_EINVAL, "NULL argument");
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = launch_build_queries(begin, end, k, nq, static_cast<SelQuery*>(qbuf), st);
  if (e == cudaSuccess) e = launch_select(values, static_cast<SelQuery*>(qbuf), nq, out, st);
  return e == cudaSuccess ? SPCN_OK : cuda_fail(e, "select_kth");
}

}  // extern "C"

// ------------------------------------------------------------------ global stats
#include "stats.h"

namespace {
// Strict + fast parameter blocks of the density coder alone (source side).
int stats_setup(const spcn_xform_params* p, int32_t white, StatsArgs& a, StrictP& sp) {
  if (!p) return fail(SPCN_EINVAL, "params is NULL");
  for (int c = 0; c < 3; ++c)
    if (!(p->src_i0[c] >= 1.0) || !std::isfinite(p->src_i0[c]))
      return fail(SPCN_EINVAL, "i0 components must be >= 1");
  int rc = check_basis(p->src_basis, "source");
  if (rc) return rc;
  if (!(p->code_lam >= 0.0)) return fail(SPCN_EINVAL, "lam must be >= 0");
  if (white < 0 || white > 255) return fail(SPCN_EINVAL, "white threshold must be in [0, 255]");
  double lut[3][256];
  od_table(p->src_i0, p->od_table, lut);
  const double one[2] = {1.0, 1.0}, i0t[3] = {255.0, 255.0, 255.0};
  fill_strict(sp, &lut[0][0], p->src_basis, p->src_basis, one, i0t, p->code_lam, p->max_sweeps);
  static thread_local FastP fp;
  const bool ok = fill_fast_scalars(fp, sp, false, fp.lut);
  a.fs = fp;
  for (int c = 0; c < 3; ++c)
    for (int i = 0; i < 256; ++i) a.lut[c][i] = static_cast<float>(lut[c][i]);
  double coef[2];
  density_error_coeffs(sp, coef);
  for (int j = 0; j < 2; ++j)   // ill-conditioned basis: every candidate goes through fp64
    a.coef[j] = ok ? std::nextafter(static_cast<float>(coef[j] * (1.0 + 2e-6)), INFINITY)
                   : INFINITY;
  a.white = static_cast<uint32_t>(white);
  // the OD table is strictly decreasing across [white, white + 1] when
  // 1 <= white < i0 (clip(x, 1, i0) grows there), so "x > white" is "OD(x) <
  // OD(white)" and the white test can run on the looked-up OD values
  bool by_od = white >= 1 && white <= 254;
  for (int c = 0; c < 3; ++c) {
    by_od = by_od && p->src_i0[c] > white && a.lut[c][white + (white < 255)] < a.lut[c][white];
    a.nwod[c] = by_od ? -a.lut[c][white] : 0.0f;
  }
  a.white_by_od = by_od ? 1u : 0u;
  return SPCN_OK;
}
// The table pass's four linear upper-bound forms (stats.cu k_stats_table):
// stain 0: u0 - a0 = (g11 t0 - g01 t1)/det - a0 and t0/g00 - a0; stain 1:
// (g00 t1 - g01 t0)/det - a1 and t1/g11 - a1, with t_j = sum_c w_cj v_c - lam,
// as k.v + b in fp64, then fp32 with the evaluation error bound added to b:
// |fp32(k.v + b) - (k.v + b)| <= 2^-21 (sum|k| V + |b|) for V = max OD (the
// fp32 table, the fp32 coefficients and three FMAs); 8x that is added.  An
// ill-conditioned basis (or no positive lower bound) makes every non-white
// pixel a candidate.
void stats_linear_forms(const StrictP& sp, const double* lo, StatsArgs& a) {
  const double g00 = sp.g00, g01 = sp.g01, g11 = sp.g11, det = sp.det, lam = sp.lam;
  double V = 0.0;
  for (int c = 0; c < 3; ++c)
    for (int x = 0; x < 256; ++x) V = std::max(V, std::fabs(sp.lut[c][x]));
  const bool ok = det > 1e-6 * g00 * g11 && g00 > 0.0 && g11 > 0.0;
  double k[4][3], b[4];
  for (int c = 0; c < 3; ++c) {
    const double w0 = sp.ws[c][0], w1 = sp.ws[c][1];
    k[0][c] = ok ? (g11 * w0 - g01 * w1) / det : 0.0;
    k[1][c] = ok ? w0 / g00 : 0.0;
    k[2][c] = ok ? (g00 * w1 - g01 * w0) / det : 0.0;
    k[3][c] = ok ? w1 / g11 : 0.0;
  }
  b[0] = ok ? (-g11 * lam + g01 * lam) / det - lo[0] : 1.0;
  b[1] = ok ? -lam / g00 - lo[0] : 1.0;
  b[2] = ok ? (-g00 * lam + g01 * lam) / det - lo[1] : 1.0;
  b[3] = ok ? -lam / g11 - lo[1] : 1.0;
  for (int i = 0; i < 4; ++i) {
    double sk = 0.0;
    for (int c = 0; c < 3; ++c) sk += std::fabs(k[i][c]);
    const double margin = 8.0 * std::ldexp(sk * V + std::fabs(b[i]), -21);
    for (int c = 0; c < 3; ++c) a.lf[i][c] = static_cast<float>(k[i][c]);
    a.lf[i][3] = std::nextafter(static_cast<float>(b[i] + margin), INFINITY);
  }
}
}  // namespace

extern "C" {

int spcn_stats_hist(const uint8_t* src, int64_t npix, const spcn_xform_params* p,
                    int32_t white_threshold, const uint32_t* base, const uint32_t* shift,
                    int32_t nbins, unsigned long long* hist, unsigned long long* counts,
                    void* stream) {
  g_err.clear();
  if (npix < 0) return fail(SPCN_EINVAL, "npix must be >= 0");
  if (nbins < 1 || nbins > 8192) return fail(SPCN_EINVAL, "nbins must be in [1, 8192]");
  if (!base || !shift || !hist || !counts) return fail(SPCN_EINVAL, "NULL argument");
  if (npix > 0 && !src) return fail(SPCN_EINVAL, "src is NULL");
  if (npix > 0 && (reinterpret_cast<uintptr_t>(src) & 15))
    return fail(SPCN_EINVAL, "src must be 16-byte aligned");
  static thread_local StatsArgs a;
  static thread_local StrictP sp;
  int rc = stats_setup(p, white_threshold, a, sp);
  if (rc) return rc;
  for (int j = 0; j < 2; ++j) {
    if (shift[j] > 23) return fail(SPCN_EINVAL, "shift must be <= 23");
    a.base[j] = base[j];
    a.shift[j] = shift[j];
    a.a[j] = a.b[j] = 0.0;
  }
  a.nbins = nbins;
  const cudaError_t e = launch_stats_hist(src, npix, a, hist, counts,
                                          static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SPCN_OK : cuda_fail(e, "stats_hist");
}

int spcn_stats_refine(const uint8_t* src, int64_t npix, const spcn_xform_params* p,
                      int32_t white_threshold, const double* lo, const double* hi,
                      unsigned long long* counts, double* cand, unsigned long long* cand_count,
                      unsigned long long cap, void* stream) {
  g_err.clear();
  if (npix < 0) return fail(SPCN_EINVAL, "npix must be >= 0");
  if (!lo || !hi || !counts || (cap > 0 && (!cand || !cand_count)))
    return fail(SPCN_EINVAL, "NULL argument");
  if (npix > 0 && !src) return fail(SPCN_EINVAL, "src is NULL");
  if (npix > 0 && (reinterpret_cast<uintptr_t>(src) & 15))
    return fail(SPCN_EINVAL, "src must be 16-byte aligned");
  static thread_local StatsArgs a;
  static thread_local StrictP sp;
  int rc = stats_setup(p, white_threshold, a, sp);
  if (rc) return rc;
  for (int j = 0; j < 2; ++j) {
    a.base[j] = 0;
    a.shift[j] = 0;
    a.a[j] = lo[j];
    a.b[j] = hi[j];
  }
  a.nbins = 1;
  const cudaError_t e = launch_stats_refine(src, npix, a, sp, counts, cand, cand_count, cap,
                                            static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SPCN_OK : cuda_fail(e, "stats_refine");
}

int spcn_stats_table(const uint8_t* src, int64_t npix, const spcn_xform_params* p,
                     int32_t white_threshold, const double* lo, unsigned long long* table,
                     unsigned long long* counts, void* stream) {
  g_err.clear();
  if (npix < 0) return fail(SPCN_EINVAL, "npix must be >= 0");
  if (!lo || !table || !counts) return fail(SPCN_EINVAL, "NULL argument");
  if (npix > 0 && !src) return fail(SPCN_EINVAL, "src is NULL");
  if (npix > 0 && (reinterpret_cast<uintptr_t>(src) & 15))
    return fail(SPCN_EINVAL, "src must be 16-byte aligned");
  static thread_local StatsArgs a;
  static thread_local StrictP sp;
  int rc = stats_setup(p, white_threshold, a, sp);
  if (rc) return rc;
  for (int j = 0; j < 2; ++j) {
    a.base[j] = 0;
    a.shift[j] = 0;
    a.a[j] = lo[j];
    a.b[j] = INFINITY;
    if (!(lo[j] > 0.0)) return fail(SPCN_EINVAL, "table pass needs lo > 0");
  }
  a.nbins = 1;
  stats_linear_forms(sp, lo, a);
  const cudaError_t e = launch_stats_table(src, npix, a, table, counts,
                                           static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SPCN_OK : cuda_fail(e, "stats_table");
}

int spcn_stats_cube_classes(const spcn_xform_params* p, int32_t white_threshold,
                            const double* lo, uint8_t* classes, void* stream) {
  g_err.clear();
  if (!lo || !classes) return fail(SPCN_EINVAL, "NULL argument");
  static thread_local StatsArgs a;
  static thread_local StrictP sp;
  int rc = stats_setup(p, white_threshold, a, sp);
  if (rc) return rc;
  for (int j = 0; j < 2; ++j)
    if (!(lo[j] > 0.0)) return fail(SPCN_EINVAL, "table pass needs lo > 0");
  stats_linear_forms(sp, lo, a);
  const cudaError_t e = launch_cube_class(a, classes, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SPCN_OK : cuda_fail(e, "stats_cube_classes");
}

int spcn_stats_table_cube(const uint8_t* src, int64_t npix, const spcn_xform_params* p,
                          int32_t white_threshold, const double* lo, const uint8_t* classes,
                          unsigned long long* table, unsigned long long* counts, void* stream) {
  g_err.clear();
  if (npix < 0) return fail(SPCN_EINVAL, "npix must be >= 0");
  if (!lo || !classes || !table || !counts) return fail(SPCN_EINVAL, "NULL argument");
  if (npix > 0 && !src) return fail(SPCN_EINVAL, "src is NULL");
  if (npix > 0 && (reinterpret_cast<uintptr_t>(src) & 15))
    return fail(SPCN_EINVAL, "src must be 16-byte aligned");
  if (reinterpret_cast<uintptr_t>(classes) & 15)
    return fail(SPCN_EINVAL, "classes must be 16-byte aligned");
  static thread_local StatsArgs a;
  static thread_local StrictP sp;
  int rc = stats_setup(p, white_threshold, a, sp);
  if (rc) return rc;
  for (int j = 0; j < 2; ++j)
    if (!(lo[j] > 0.0)) return fail(SPCN_EINVAL, "table pass needs lo > 0");
  stats_linear_forms(sp, lo, a);
  const cudaError_t e = launch_stats_cube(src, npix, a, classes, table, counts,
                                          static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SPCN_OK : cuda_fail(e, "stats_table_cube");
}

int spcn_table_entries_hist(const double* x, const unsigned long long* w, int64_t m,
                            const double* lo, const double* scale, int32_t nbins,
                            unsigned long long* hist, void* stream) {
  g_err.clear();
  if (m < 0) return fail(SPCN_EINVAL, "m must be >= 0");
  if (nbins < 1 || nbins > 8192) return fail(SPCN_EINVAL, "nbins must be in [1, 8192]");
  if (!lo || !scale || !hist || (m > 0 && (!x || !w))) return fail(SPCN_EINVAL, "NULL argument");
  for (int j = 0; j < 2; ++j)
    if (!(scale[j] >= 0.0) || !std::isfinite(scale[j]) || !std::isfinite(lo[j]))
      return fail(SPCN_EINVAL, "lo/scale must be finite, scale >= 0");
  const cudaError_t e = launch_entries_hist(x, w, m, lo, scale, nbins, hist,
                                            static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SPCN_OK : cuda_fail(e, "table_entries_hist");
}

int spcn_table_entries_collect(const double* x, const unsigned long long* w, int64_t m,
                               const double* lo, const double* scale, int32_t nbins,
                               const int32_t* bins, double* vals, unsigned long long* wts,
                               unsigned long long cap, unsigned long long* nsel, void* stream) {
  g_err.clear();
  if (m < 0) return fail(SPCN_EINVAL, "m must be >= 0");
  if (nbins < 1 || nbins > 8192) return fail(SPCN_EINVAL, "nbins must be in [1, 8192]");
  if (!lo || !scale || !bins || !nsel || (m > 0 && (!x || !w)) || (cap > 0 && (!vals || !wts)))
    return fail(SPCN_EINVAL, "NULL argument");
  const cudaError_t e = launch_entries_collect(x, w, m, lo, scale, nbins, bins, vals, wts, cap,
                                               nsel, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SPCN_OK : cuda_fail(e, "table_entries_collect");
}

int spcn_stats_table_scan(const spcn_xform_params* p, const unsigned long long* table,
                          double* x, unsigned long long* w, unsigned long long cap,
                          unsigned long long* n_out, void* stream) {
  g_err.clear();
  if (!table || !n_out || (cap > 0 && (!x || !w))) return fail(SPCN_EINVAL, "NULL argument");
  static thread_local StatsArgs a;
  static thread_local StrictP sp;
  int rc = stats_setup(p, 220, a, sp);
  if (rc) return rc;
  const cudaError_t e = launch_table_scan(table, sp, x, w, cap, n_out,
                                          static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SPCN_OK : cuda_fail(e, "stats_table_scan");
}

}  // extern "C"

// ------------------------------------------------------------------ synthetic input
#include "synth.h"

// ------------------------------------------------------------------ small read-backs
namespace {
__global__ void k_copy_to_host(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst,
                               int64_t words) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < words;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}
}  // namespace

// Device -> pinned host through the SMs (stores over PCIe into the mapped
// allocation) instead of a copy engine: a read-back of a few KB never queues
// behind multi-hundred-MB transfers another stream has on the copy engine.
extern "C" int spcn_fit_sample_step(const uint8_t* img, const spcn_patch* patches, int32_t n,
                                    int32_t max_chunks, int32_t k0, const int32_t* dims,
                                    const spcn_visit_plan* plan, int32_t white_threshold,
                                    int32_t zero_arena, void* arena_a, int32_t* counts,
                                    spcn_patch_take* takes, uint8_t* sample_out,
                                    void* readback_pinned, int64_t readback_bytes, void* stream) {
  g_err.clear();
  if (!arena_a || !readback_pinned || readback_bytes < 0 || readback_bytes > SPCN_FIT_ARENA_A)
    return fail(SPCN_EINVAL, "bad arena / readback");
  char* A = static_cast<char*>(arena_a);
  int64_t* state = reinterpret_cast<int64_t*>(A);
  int64_t* offsets = reinterpret_cast<int64_t*>(A + 64);
  double* i0 = reinterpret_cast<double*>(A + 80);
  int32_t* empty = reinterpret_cast<int32_t*>(A + 104);
  int32_t* hist = reinterpret_cast<int32_t*>(A + 128);
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (zero_arena) {
    const cudaError_t e = cudaMemsetAsync(arena_a, 0, SPCN_FIT_ARENA_A, st);
    if (e != cudaSuccess) return cuda_fail(e, "memset");
  }
  int rc = spcn_sample_count(img, patches, n, max_chunks, white_threshold, counts, stream);
  if (!rc) rc = spcn_sample_visit(counts, n, max_chunks, k0, dims, plan, state, takes, offsets,
                                  stream);
  if (!rc) rc = spcn_sample_compact(img, patches, n, max_chunks, white_threshold, counts, takes,
                                    sample_out, hist, stream);
  if (!rc) rc = spcn_i0_from_hist(hist, 1, i0, empty, stream);
  if (!rc) rc = spcn_readback(arena_a, readback_pinned, readback_bytes, stream);
  return rc;
}

extern "C" int spcn_fit_basis_step(const uint8_t* sample, int64_t m, const int64_t* offsets,
                                   const double* lut_pinned, double* lut_dev,
                                   const spcn_snmf_cfg* cfg, double* hscratch, double* history,
                                   void* arena_b, double code_lam, int32_t max_sweeps, double* h,
                                   void* qbuf, double* selbuf, int32_t want_p99,
                                   void* readback_pinned, int64_t readback_bytes, void* stream) {
  g_err.clear();
  if (!arena_b || !lut_pinned || !lut_dev || !readback_pinned || readback_bytes < 0 ||
      readback_bytes > SPCN_FIT_ARENA_B)
    return fail(SPCN_EINVAL, "bad arena / table / readback");
  char* B = static_cast<char*>(arena_b);
  double* basis = reinterpret_cast<double*>(B);
  double* p99 = reinterpret_cast<double*>(B + 48);
  int32_t* info = reinterpret_cast<int32_t*>(B + 64);
  int32_t* absent = reinterpret_cast<int32_t*>(B + 80);
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  const cudaError_t e =
      cudaMemcpyAsync(lut_dev, lut_pinned, 768 * sizeof(double), cudaMemcpyHostToDevice, st);
  if (e != cudaSuccess) return cuda_fail(e, "od table upload");
  int rc = spcn_snmf_batched(sample, nullptr, offsets, 1, lut_dev, cfg, hscratch, m, basis, history,
                             info, stream);
  if (!rc) rc = spcn_code_samples(sample, offsets, 1, m, lut_dev, basis, code_lam, max_sweeps, h, m,
                                  stream);
  if (!rc && want_p99)
    rc = spcn_percentile_segments(h, m, offsets, 1, 99.0, qbuf, selbuf, p99, absent, stream);
  if (!rc) rc = spcn_readback(arena_b, readback_pinned, readback_bytes, stream);
  return rc;
}

extern "C" int spcn_stream_sync(void* stream) {
  g_err.clear();
  const cudaError_t e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SPCN_OK : cuda_fail(e, "stream_sync");
}

extern "C" int spcn_readback(const void* src, void* host_pinned, int64_t bytes, void* stream) {
  g_err.clear();
  if (bytes < 0) return fail(SPCN_EINVAL, "bytes must be >= 0");
  if (bytes == 0) return SPCN_OK;
  if (!src || !host_pinned) return fail(SPCN_EINVAL, "NULL argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  void* dptr = nullptr;
  const bool aligned = ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(host_pinned) |
                         static_cast<uintptr_t>(bytes)) & 3) == 0;
  if (aligned && cudaHostGetDevicePointer(&dptr, host_pinned, 0) == cudaSuccess && dptr) {
    const int64_t words = bytes / 4;
    int grid = static_cast<int>((words + 255) / 256);
    if (grid > 64) grid = 64;
    k_copy_to_host<<<grid, 256, 0, st>>>(static_cast<const uint32_t*>(src),
                                         static_cast<uint32_t*>(dptr), words);
    const cudaError_t e = launched();
    return e == cudaSuccess ? SPCN_OK : cuda_fail(e, "readback");
  }
  cudaGetLastError();   // not mapped / unaligned: plain async copy
  const cudaError_t e = cudaMemcpyAsync(host_pinned, src, bytes, cudaMemcpyDeviceToHost, st);
  return e == cudaSuccess ? SPCN_OK : cuda_fail(e, "readback");
}

extern "C" int spcn_render_synthetic(uint8_t* out, int64_t width, int64_t row0, int64_t rows,
                                     int64_t height, uint64_t seed, const spcn_synth_params* p,
                                     void* stream) {
  g_err.clear();
  if (!p) return fail(SPCN_EINVAL, "params is NULL");
  if (width < 1 || rows < 0 || row0 < 0 || row0 + rows > height)
    return fail(SPCN_EINVAL, "bad slide geometry");
  if (rows == 0) return SPCN_OK;
  if (!out) return fail(SPCN_EINVAL, "out is NULL");
  if ((reinterpret_cast<uintptr_t>(out) & 15u) != 0)
    return fail(SPCN_EINVAL, "out must be 16-byte aligned");
  cudaError_t e = launch_render(out, width, row0, rows, height, seed, *p,
                                static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SPCN_OK : cuda_fail(e, "render_synthetic");
}

// ------------------------------------------------------------------ batched recolouring
#include "batch.h"

extern "C" {

int spcn_batch_sizes(size_t* fast_scalar_bytes, size_t* strict_param_bytes) {
  if (fast_scalar_bytes) *fast_scalar_bytes = sizeof(FastS);
  if (strict_param_bytes) *strict_param_bytes = sizeof(StrictP);
  return SPCN_OK;
}

int spcn_batch_params(int32_t nitems, const double* i0, const double* luts, const double* bases,
                      const double* p99, const spcn_batch_target* tgt, double code_lam,
                      int32_t max_sweeps, int32_t precision, void* fast_scalars, float* flut,
                      void* strict_params, int32_t* status, void* stream) {
  g_err.clear();
  if (nitems < 0) return fail(SPCN_EINVAL, "nitems must be >= 0");
  if (!tgt) return fail(SPCN_EINVAL, "target is NULL");
  int rc = check_basis(tgt->basis, "target");
  if (rc) return rc;
  if (!(code_lam >= 0.0)) return fail(SPCN_EINVAL, "lam must be >= 0");
  if (precision < 0 || precision > 2) return fail(SPCN_EINVAL, "unknown precision");
  if (nitems == 0) return SPCN_OK;
  if (!i0 || !luts || !bases || !p99 || !fast_scalars || !flut || !strict_params || !status)
    return fail(SPCN_EINVAL, "NULL argument");
  BatchTarget t;
  for (int c = 0; c < 3; ++c) t.i0[c] = tgt->i0[c];
  for (int k = 0; k < 6; ++k) t.basis[k] = tgt->basis[k];
  t.p99[0] = tgt->p99[0];
  t.p99[1] = tgt->p99[1];
  cudaError_t e = launch_build_params(nitems, i0, luts, bases, p99, t, code_lam, max_sweeps,
                                      precision == SPCN_PREC_EXACT ? 1 : 0,
                                      static_cast<FastS*>(fast_scalars), flut,
                                      static_cast<StrictP*>(strict_params), status,
                                      static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? SPCN_OK : cuda_fail(e, "batch_params");
}

int spcn_xform_batch(const uint8_t* src, uint8_t* dst, int32_t nitems, const int64_t* off_host,
                     const int64_t* off_dev, const void* fast_scalars, const int32_t* status_host,
                     const int32_t* status_dev, const float* flut, const void* strict_params,
                     int32_t precision, void* workspace, size_t workspace_bytes, void* stream) {
  g_err.clear();
  if (nitems < 0) return fail(SPCN_EINVAL, "nitems must be >= 0");
  if (nitems == 0) return SPCN_OK;
  if (!src || !dst || !off_host || !off_dev || !fast_scalars || !status_host || !status_dev ||
      !flut || !strict_params)
    return fail(SPCN_EINVAL, "NULL argument");
  if (precision < 0 || precision > 2) return fail(SPCN_EINVAL, "unknown precision");
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  const FastS* fs = static_cast<const FastS*>(fast_scalars);
  const StrictP* sps = static_cast<const StrictP*>(strict_params);
  const bool strict_all = precision == SPCN_PREC_STRICT;
  const bool exact = precision == SPCN_PREC_EXACT;
  int64_t max_pix = 0;
  bool any_strict = false, any_fast = false;
  for (int i = 0; i < nitems; ++i) {
    const int64_t n = off_host[i + 1] - off_host[i];
    if (n < 0) return fail(SPCN_EINVAL, "offsets must be non-decreasing");
    if ((off_host[i] & 15) != 0 || (n & 15) != 0)
      return fail(SPCN_EINVAL, "item pixel offsets and sizes must be multiples of 16");
    max_pix = n > max_pix ? n : max_pix;
    any_strict = any_strict || status_host[i] == 1 || (strict_all && status_host[i] == 0);
    any_fast = any_fast || status_host[i] == 0;
  }
  if ((reinterpret_cast<uintptr_t>(src) & 15) || (reinterpret_cast<uintptr_t>(dst) & 15))
    return fail(SPCN_EINVAL, "src/dst must be 16-byte aligned");
  cudaError_t e = cudaSuccess;
  // EXACT: workspace = [per-CTA counters][per-item segments][per-CTA lists]
  BatchRepair br{nullptr, nullptr, 0, nullptr};
  if (exact) {
    const size_t grid = static_cast<size_t>(batch_grid(nitems));
    const size_t head = 8 * grid + 24 * static_cast<size_t>(nitems);
    if (!workspace || workspace_bytes < head + 8 * grid)
      return fail(SPCN_EINVAL, "EXACT precision needs a workspace");
    br.counts = static_cast<unsigned long long*>(workspace);
    br.seg = br.counts + grid;
    br.items = br.seg + 3 * static_cast<size_t>(nitems);
    br.cap_cta = (workspace_bytes - head) / 8 / grid;
    if ((e = cudaMemsetAsync(br.counts, 0, 8 * grid, st)) != cudaSuccess)
      return cuda_fail(e, "memset");
  }
  if (!strict_all && any_fast) {
    // one persistent launch over every fast-path item (status 0)
    e = launch_xform_batch(exact ? 0 : 1, src, dst, nitems, off_dev, status_dev, fs, flut, br, st);
    if (e != cudaSuccess) return cuda_fail(e, "xform_batch");
    if (exact && (e = launch_repair_items(src, dst, sps, off_dev, status_dev, nitems, br, st)) !=
                     cudaSuccess)
      return cuda_fail(e, "repair_items");
  }
  if (any_strict) {
    // strict items: status 1 (or every valid item in STRICT precision)
    e = launch_strict_batch(src, dst, sps, off_dev, status_dev, nitems, max_pix, st);
    if (e != cudaSuccess) return cuda_fail(e, "strict_batch");
  }
  return SPCN_OK;
}

}  // extern "C"

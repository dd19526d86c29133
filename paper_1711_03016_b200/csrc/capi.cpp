// C ABI (include/dlvm.h) and the run-time executor.
//
// dlvm_fn_create = the NNKit JIT phases of PAPER.md §3.4 L386-390 for one
// shape-specialised function: parse (.dl text, Fig. 3 syntax) -> verify
// (Fig. 2 "Analyses & Verification") -> differentiate the gradient
// declaration by adjoint code generation (§3.1.3) -> dead-code
// elimination (L304-305) -> plan fused sm_100a launches.  dlvm_fn_run /
// dlvm_grad_run bind caller pointers and enqueue the planned launches on the
// caller's stream: no allocation, no host synchronisation (graph-capturable).
#include <nvtx3/nvToolsExt.h>
#include <cuda_runtime.h>

#include <cstring>
#include <new>
#include <optional>
#include <sstream>
#include <string>

#include "../../include/dlvm.h"
#include "ir.h"
#include "jit.h"
#include "kernels/kernels.h"
#include "kernels/spec_registry.h"
#include "plan.h"

using namespace dlvm;

struct dlvm_fn_s {
  Function primal;
  std::optional<Function> grad;
  Function opt_primal;           // what the plans execute (optimize_function unless DLVM_NO_OPT)
  std::optional<Function> opt_grad;
  Plan plan[2];
  bool planned[2] = {false, false};
  std::string plan_error[2];
  dlvm_options opts{};
  int n_grads = 0;
  std::vector<void*> launch_events[2];
  bool specialize = true;
  std::vector<void*> jit_fn[2];  // per plan step: create-time specialised kernel (CUfunction) or null
  std::vector<char> out_read[2]; // per output: some launch reads it back (it cannot be bound as DLVM_F32_ADD)
  // two-stream schedule (plan_streams): per step the stream (0 = caller's,
  // 1 = the handle's auxiliary stream), the earlier steps on the other
  // stream it waits for, and whether an event is recorded after it
  std::vector<char> step_stream[2];
  std::vector<std::vector<int>> step_waits[2];
  std::vector<char> step_signals[2];
  bool concurrent[2] = {false, false};
  int device = -1;
  cudaStream_t aux = nullptr;
  std::vector<cudaEvent_t> events;  // one per step that signals, plus fork / join
  ~dlvm_fn_s() {
    for (cudaEvent_t e : events) cudaEventDestroy(e);
    if (aux) cudaStreamDestroy(aux);
  }
  std::string jit_report;        // print mode 8
};

namespace {

thread_local std::string g_last_error;

int64_t numel_of(const dlvm_tensor& t) {
  int64_t n = 1;
  for (int d = 0; d < t.rank; ++d) n *= t.shape[d];
  return n;
}

// buffers a step reads / writes (buffer ids of the plan)
void step_buffers(const Step& st, std::vector<int>* rd, std::vector<int>* wr) {
  auto group = [&](const EwGroup& g) {
    for (auto& r : g.inputs)
      if (r.buf >= 0) rd->push_back(r.buf);
    for (auto& r : g.stores) wr->push_back(r.buf);
    for (auto& r : g.reduces) {
      if (r.buf >= 0) wr->push_back(r.buf);
      if (r.direct_buf >= 0) wr->push_back(r.direct_buf);
    }
  };
  if (st.kind == Step::EW) {
    group(st.ew);
  } else if (st.kind == Step::GEMM) {
    for (auto& sg : st.gemm.seg) {
      rd->push_back(sg.a.buf);
      rd->push_back(sg.b.buf);
    }
    group(st.gemm.epi);
  } else if (st.kind == Step::CAST) {
    wr->push_back(st.cast.dst_buf);
  }
}

// Two-stream schedule of a plan: a tensor-core GEMM that does not depend
// (through any buffer, transitively) on the GEMM launched before it runs on
// the auxiliary stream beside it -- the independent weight- and activation-
// gradient GEMMs of a layer (dW_l = H^T dZ_l and dZ_{l-1} = dZ_l W^T) -- and
// the steps that only need it follow it there; every cross-stream
// dependency becomes an event wait.  Both GEMMs of such a pair use dynamic
// tile scheduling, so the one that starts second takes over tiles as the
// other's SMs free up.
void plan_streams(dlvm_fn_s* h, int which) {
  const Plan& P = h->plan[which];
  const int n = (int)P.steps.size();
  std::vector<std::vector<int>> rd(n), wr(n), deps(n);
  for (int i = 0; i < n; ++i) step_buffers(P.steps[i], &rd[i], &wr[i]);
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < j; ++i) {
      bool d = false;
      for (int b : rd[j])
        for (int c : wr[i]) d |= b == c;   // RAW
      for (int b : wr[j]) {
        for (int c : wr[i]) d |= b == c;   // WAW
        for (int c : rd[i]) d |= b == c;   // WAR
      }
      if (d) deps[j].push_back(i);
    }
  // ancestors (transitive dependencies) as bit rows
  std::vector<std::vector<char>> anc(n, std::vector<char>(n, 0));
  for (int j = 0; j < n; ++j)
    for (int i : deps[j]) {
      anc[j][i] = 1;
      for (int k = 0; k < n; ++k) anc[j][k] |= anc[i][k];
    }
  std::vector<char>& stream = h->step_stream[which];
  stream.assign(n, 0);
  int prev_gemm = -1;
  bool any = false;
  for (int j = 0; j < n; ++j) {
    const Step& s = P.steps[j];
    if (s.kind == Step::GEMM && s.gemm.tensor_core) {
      if (prev_gemm >= 0 && stream[prev_gemm] == 0 && !anc[j][prev_gemm]) {
        stream[j] = 1;
        any = true;
      }
      prev_gemm = j;
    } else if (s.kind == Step::EVENT) {
      // recorded on the stream of the gradient's last writer (the step before)
      stream[j] = j > 0 ? stream[j - 1] : 0;
    } else {
      // element-wise steps follow their latest dependency
      int last = -1;
      for (int i : deps[j]) last = std::max(last, i);
      stream[j] = last >= 0 ? stream[last] : 0;
    }
  }
  h->concurrent[which] = any;
  std::vector<std::vector<int>>& waits = h->step_waits[which];
  std::vector<char>& signals = h->step_signals[which];
  waits.assign(n, {});
  signals.assign(n, 0);
  if (!any) return;
  for (int j = 0; j < n; ++j) {
    // wait for the latest dependency on the other stream (earlier ones on it
    // are ordered by that stream)
    int last = -1;
    for (int i : deps[j])
      if (stream[i] != stream[j]) last = std::max(last, i);
    if (P.steps[j].kind == Step::EVENT && j > 0 && stream[j - 1] != stream[j]) last = j - 1;
    if (last >= 0) {
      waits[j].push_back(last);
      signals[last] = 1;
    }
  }
}

// outputs whose buffer a later launch of the plan reads (e.g. a kept value
// feeding more work): their final value must be stored, not accumulated
std::vector<char> outputs_read(const Plan& P) {
  std::vector<char> read(P.n_outputs, 0);
  auto mark = [&](int buf) {
    if (buf >= 0 && buf < (int)P.bufs.size() && P.bufs[buf].kind == BufferSlot::Output) read[P.bufs[buf].index] = 1;
  };
  for (const Step& st : P.steps) {
    if (st.kind == Step::EW) {
      for (auto& r : st.ew.inputs) mark(r.buf);
    } else if (st.kind == Step::GEMM) {
      for (auto& sg : st.gemm.seg) {
        mark(sg.a.buf);
        mark(sg.b.buf);
      }
      for (auto& r : st.gemm.epi.inputs) mark(r.buf);
    }
  }
  return read;
}

dlvm_status fail(dlvm_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

dlvm_status from_error(const Error& e) {
  g_last_error = e.what();
  return (dlvm_status)e.status;
}

void fill_sig(const Type& t, dlvm_tensor* out) {
  std::memset(out, 0, sizeof(*out));
  out->data = nullptr;
  out->dtype = t.dtype == DType::Bool ? DLVM_BOOL : t.dtype == DType::F64 ? DLVM_F64 : DLVM_F32;
  out->rank = t.rank();
  for (int i = 0; i < t.rank() && i < DLVM_MAX_RANK; ++i) out->shape[i] = t.shape[i];
}

bool shape_matches(const dlvm_tensor& t, const Type& ty) {
  if (t.rank != ty.rank()) return false;
  for (int i = 0; i < t.rank; ++i)
    if (t.shape[i] != ty.shape[i]) return false;
  return true;
}

SType stype_of(int32_t dt) {
  return dt == DLVM_BF16 ? SType::BF16 : dt == DLVM_BOOL ? SType::U8 : dt == DLVM_F32_ADD ? SType::F32_ADD : SType::F32;
}

struct Bound {
  std::vector<void*> ptr;     // per BufferSlot
  std::vector<uint8_t> st;    // runtime storage type per BufferSlot
};

void to_dev(const EwGroup& g, const Bound& b, EwParams* p) {
  std::memset(p, 0, sizeof(*p));
  p->ndims = g.ndims;
  p->ncols = g.ncols;
  p->vec = g.vec;
  p->rpt = g.rpt;
  for (int d = 0; d < kMaxIterDims; ++d) p->dims[d] = g.dims[d];
  p->gx = g.gx;
  p->gy = g.gy;
  p->prog = g.prog;
  for (size_t i = 0; i < g.inputs.size(); ++i) {
    const IterRef& r = g.inputs[i];
    EwDevIn& d = p->in[i];
    if (r.buf < 0) continue;  // accumulator
    const uint8_t st = b.st[r.buf];
    size_t esz = (size_t)st_bytes(st);
    d.ptr = static_cast<const char*>(b.ptr[r.buf]) + r.offset * esz;
    for (int k = 0; k < kMaxIterDims; ++k) d.s[k] = r.strides[k];
    d.nchunks = r.nchunks;
    d.chunk_stride = r.chunk_stride;
    d.chunk_op = r.chunk_op;
    d.st = st;
  }
  for (size_t i = 0; i < g.stores.size(); ++i) {
    const IterRef& r = g.stores[i];
    EwDevOut& d = p->out[i];
    const uint8_t st = b.st[r.buf];
    size_t esz = (size_t)st_bytes(st);
    d.ptr = static_cast<char*>(b.ptr[r.buf]) + r.offset * esz;
    for (int k = 0; k < kMaxIterDims; ++k) d.s[k] = r.strides[k];
    d.st = st;
  }
  for (size_t i = 0; i < g.reduces.size(); ++i) {
    const int hb = g.reduces[i].direct_buf;
    const bool direct = hb >= 0 && b.st[hb] == (uint8_t)SType::F32;
    p->red[i] = static_cast<float*>(b.ptr[direct ? hb : g.reduces[i].buf]);
  }
}

// epilogue vectorisation along n: every ref must allow 4-wide access
// Coarse filter for the tcgen05 epilogue's vector path (contiguous rows,
// 16-byte base pointers); the kernel additionally checks, per tile row, that
// each row start is aligned to the vector width it uses (a u8 row of 1000
// elements is 8-byte aligned on odd rows).
int epi_vec(const EwParams& e) {
  for (int i = 1; i < e.prog.n_in; ++i) {
    const EwDevIn& r = e.in[i];
    if (r.nchunks != 1) return 1;
    if (r.s[1] != 0 && r.s[1] != 1) return 1;
    if (r.s[1] == 1 && (r.s[0] % 4 || (reinterpret_cast<uintptr_t>(r.ptr) % 16))) return 1;
  }
  for (int i = 0; i < e.prog.n_stores; ++i) {
    const EwDevOut& r = e.out[i];
    if (r.s[1] != 1 || r.s[0] % 4 || (reinterpret_cast<uintptr_t>(r.ptr) % 16)) return 1;
  }
  return 4;
}

struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

struct DeviceGuard {
  int prev = -1;
  cudaError_t set(int dev) {
    cudaError_t e = cudaGetDevice(&prev);
    if (e != cudaSuccess) return e;
    if (prev == dev) {
      prev = -1;
      return cudaSuccess;
    }
    return cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

dlvm_status execute(dlvm_fn fn, int which, const dlvm_tensor* in, int n_in, const dlvm_tensor* seed,
                    dlvm_tensor* out, int n_out, void* workspace, void* stream_v, void* const* events) {
  if (!fn) return fail(DLVM_ERR_USAGE, "NULL handle");
  if (fn->opts.flags & DLVM_PLAN_ONLY) return fail(DLVM_ERR_USAGE, "handle was created with DLVM_PLAN_ONLY");
  if (!fn->planned[which]) return fail(DLVM_ERR_UNSUPPORTED, fn->plan_error[which]);
  const Function& f = which ? *fn->grad : fn->primal;
  const Plan& P = fn->plan[which];
  if (n_in != P.n_inputs) return fail(DLVM_ERR_USAGE, "expected " + std::to_string(P.n_inputs) + " inputs");
  if (n_out != P.n_outputs) return fail(DLVM_ERR_USAGE, "expected " + std::to_string(P.n_outputs) + " outputs");
  if (n_in && !in) return fail(DLVM_ERR_USAGE, "NULL inputs");
  if (n_out && !out) return fail(DLVM_ERR_USAGE, "NULL outputs");
  if (P.seed_is_input && !seed) return fail(DLVM_ERR_USAGE, "seedable gradient needs a seed");
  if (!P.seed_is_input && seed) return fail(DLVM_ERR_USAGE, "seed given for a non-seedable gradient");
  if (P.workspace_bytes && !workspace) return fail(DLVM_ERR_USAGE, "NULL workspace");
  if (reinterpret_cast<uintptr_t>(workspace) % 256) return fail(DLVM_ERR_USAGE, "workspace must be 256-byte aligned");
  for (int i = 0; i < n_in; ++i) {
    const Type& t = f.params[i];
    if (!shape_matches(in[i], t)) return fail(DLVM_ERR_USAGE, "input " + std::to_string(i) + " shape mismatch");
    bool ok = t.dtype == DType::Bool ? in[i].dtype == DLVM_BOOL
                                     : (in[i].dtype == DLVM_F32 || (in[i].dtype == DLVM_BF16 && P.input_bf16_ok[i]) ||
                                        (in[i].dtype == DLVM_BOOL && P.input_u8_ok[i]));
    if (!ok) return fail(DLVM_ERR_USAGE, "input " + std::to_string(i) + " dtype mismatch");
    if (!in[i].data || reinterpret_cast<uintptr_t>(in[i].data) % 16)
      return fail(DLVM_ERR_USAGE, "input " + std::to_string(i) + " NULL or not 16-byte aligned");
  }
  if (seed) {
    const Type& t = f.params.back();
    if (!shape_matches(*seed, t) || seed->dtype != DLVM_F32 || !seed->data ||
        reinterpret_cast<uintptr_t>(seed->data) % 16)
      return fail(DLVM_ERR_USAGE, "seed must be f32, 16-byte aligned, of type " + t.str());
  }
  for (int i = 0; i < n_out; ++i) {
    const Type& t = f.results[i];
    if (!shape_matches(out[i], t)) return fail(DLVM_ERR_USAGE, "output " + std::to_string(i) + " shape mismatch");
    bool ok = t.dtype == DType::Bool ? out[i].dtype == DLVM_BOOL
                                     : (out[i].dtype == DLVM_F32 || out[i].dtype == DLVM_BF16 || out[i].dtype == DLVM_F32_ADD);
    if (!ok) return fail(DLVM_ERR_USAGE, "output " + std::to_string(i) + " dtype mismatch");
    if (out[i].dtype == DLVM_F32_ADD && fn->out_read[which][i])
      return fail(DLVM_ERR_USAGE, "output " + std::to_string(i) + " is read by a later launch: it cannot be accumulated");
    if (!out[i].data || reinterpret_cast<uintptr_t>(out[i].data) % 16)
      return fail(DLVM_ERR_USAGE, "output " + std::to_string(i) + " NULL or not 16-byte aligned");
  }
  cudaStream_t stream_main = static_cast<cudaStream_t>(stream_v);
  cudaStream_t stream = stream_main;
  // dlvm_options.device >= 0: the launches go to that device (made current
  // for the duration of the call, then restored); -1: the caller's current one
  DeviceGuard dg;
  if (fn->opts.device >= 0) {
    cudaError_t e = dg.set(fn->opts.device);
    if (e != cudaSuccess) return fail(DLVM_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  }
  // parameter i of the function: an input, or the seed (last parameter of a
  // seedable gradient, passed separately; it may feed a dot and need a cast)
  auto param = [&](int i) -> const dlvm_tensor& { return i < n_in ? in[i] : *seed; };
  Bound b;
  b.ptr.resize(P.bufs.size());
  b.st.resize(P.bufs.size());
  for (size_t k = 0; k < P.bufs.size(); ++k) {
    const BufferSlot& s = P.bufs[k];
    b.st[k] = (uint8_t)s.st;
    switch (s.kind) {
      case BufferSlot::Input:
        b.ptr[k] = in[s.index].data;
        b.st[k] = (uint8_t)stype_of(in[s.index].dtype);
        break;
      case BufferSlot::Output:
        b.ptr[k] = out[s.index].data;
        b.st[k] = (uint8_t)stype_of(out[s.index].dtype);
        break;
      case BufferSlot::Seed:
        b.ptr[k] = seed->data;
        break;
      case BufferSlot::Work:
        if (s.cast_of >= 0 && param(s.cast_of).dtype == DLVM_BF16 && s.cast_ld == 0)
          b.ptr[k] = param(s.cast_of).data;
        else
          b.ptr[k] = static_cast<char*>(workspace) + s.offset;
        break;
    }
  }
  const std::vector<void*>& lev = fn->launch_events[which];
  int li = 0;
  auto mark = [&](int i) -> cudaError_t {
    if (lev.empty() || !lev[i]) return cudaSuccess;
    return cudaEventRecord(static_cast<cudaEvent_t>(lev[i]), stream);
  };
  const std::vector<void*>& jit = fn->jit_fn[which];
  // dynamic tile scheduling of the tcgen05 GEMMs (DLVM_GEMM_DYN=1): their
  // work counters live in the workspace and start at zero every run
  static const bool dyn_env = [] {
    const char* e = std::getenv("DLVM_GEMM_DYN");
    return e && e[0] == '1';
  }();
  // two streams (plan_streams) when enabled (DLVM_CONCURRENT=1), no
  // profiling hook is set and no output overlaps an input in memory (the
  // schedule's dependencies are by buffer, not by address).  Off by default:
  // measured on c3 (tools/gemm_trace.py), the GEMM started second gets only
  // the SMs the first one leaves idle until that one's single-tile CTAs
  // exit, so the pair takes as long as the two in sequence (d13 || d11:
  // 44.5 vs 35.4 us; d20 || d18: 85 vs 81 us) -- each CTA still pays its own
  // prologue and exposed epilogue.
  static const bool conc_env = [] {
    const char* e = std::getenv("DLVM_CONCURRENT");
    return e && e[0] == '1';
  }();
  bool conc = conc_env && fn->concurrent[which] && lev.empty();
  for (size_t k = 0; conc && k < P.bufs.size(); ++k) {
    if (P.bufs[k].kind != BufferSlot::Output) continue;
    const dlvm_tensor& o = out[P.bufs[k].index];
    const char* o0 = static_cast<const char*>(o.data);
    const char* o1 = o0 + numel_of(o) * st_bytes((uint8_t)stype_of(o.dtype));
    for (int i = 0; i < n_in && conc; ++i) {
      const char* i0 = static_cast<const char*>(in[i].data);
      const char* i1 = i0 + numel_of(in[i]) * st_bytes((uint8_t)stype_of(in[i].dtype));
      conc = !(o0 < i1 && i0 < o1);
    }
  }
  const int nsteps = (int)P.steps.size();
  if (conc) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (!fn->aux || fn->device != dev) {
      if (fn->aux) cudaStreamDestroy(fn->aux);
      for (cudaEvent_t ev : fn->events) cudaEventDestroy(ev);
      fn->events.clear();
      fn->aux = nullptr;
      if (cudaStreamCreateWithFlags(&fn->aux, cudaStreamNonBlocking) != cudaSuccess)
        return fail(DLVM_ERR_CUDA, "cudaStreamCreate failed");
      fn->device = dev;
    }
    while ((int)fn->events.size() < nsteps + 1) {
      cudaEvent_t ev;
      if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess)
        return fail(DLVM_ERR_CUDA, "cudaEventCreate failed");
      fn->events.push_back(ev);
    }
    // fork: the auxiliary stream starts after everything queued before this run
    cudaError_t e = cudaEventRecord(fn->events[nsteps], stream_main);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(fn->aux, fn->events[nsteps], 0);
    if (e != cudaSuccess) return fail(DLVM_ERR_CUDA, std::string("fork: ") + cudaGetErrorString(e));
  }
  // dynamic tile scheduling (DLVM_GEMM_DYN=1, or every GEMM of a two-stream
  // run): the work counters live in the workspace and start at zero
  const bool dyn = (dyn_env || conc) && P.sched_buf >= 0;
  const bool hyb = !dyn && P.hybrid_counters && P.sched_buf >= 0 && gemm_hybrid_enabled();  // multicast + pair
  if (dyn || hyb) {
    cudaError_t e = cudaMemsetAsync(b.ptr[P.sched_buf], 0, (size_t)P.n_sched * 8, stream_main);
    if (e != cudaSuccess) return fail(DLVM_ERR_CUDA, std::string("cudaMemsetAsync: ") + cudaGetErrorString(e));
  }
  bool aux_used = false;
  static const bool split_red_env = [] {
    const char* e = std::getenv("DLVM_GEMM_SPLITRED");
    return !(e && e[0] == '0');
  }();
  int red_skip = -1;
  for (size_t si = 0; si < P.steps.size(); ++si) {
    const Step& st = P.steps[si];
    void* const jf = si < jit.size() ? jit[si] : nullptr;
    cudaError_t e = cudaSuccess;
    if (conc) {
      stream = fn->step_stream[which][si] ? fn->aux : stream_main;
      aux_used |= stream == fn->aux;
      for (int w : fn->step_waits[which][si])
        if ((e = cudaStreamWaitEvent(stream, fn->events[w], 0)) != cudaSuccess)
          return fail(DLVM_ERR_CUDA, std::string("cudaStreamWaitEvent: ") + cudaGetErrorString(e));
    }
    // steps with nothing to do in this binding: a finalize whose producer
    // wrote the single partial into the f32 home, and the sum of K-split
    // partials that the GEMM added into the f32 home itself (split_red)
    if ((st.kind == Step::EW && st.ew.finalize && st.ew.direct_buf >= 0 && b.st[st.ew.direct_buf] == (uint8_t)SType::F32) ||
        (int)si == red_skip) {
      if (st.counted_launch() && (e = mark(li++)) != cudaSuccess)  // an empty interval keeps the events aligned
        return fail(DLVM_ERR_CUDA, std::string("cudaEventRecord: ") + cudaGetErrorString(e));
      if (conc && fn->step_signals[which][si] && (e = cudaEventRecord(fn->events[si], stream)) != cudaSuccess)
        return fail(DLVM_ERR_CUDA, std::string("cudaEventRecord: ") + cudaGetErrorString(e));
      continue;
    }
    if (st.counted_launch() && (e = mark(li++)) != cudaSuccess)
      return fail(DLVM_ERR_CUDA, std::string("cudaEventRecord: ") + cudaGetErrorString(e));
    // one NVTX range per launch group, named by the plan step
    // ("gemm tcgen05 bf16 %z1 M=..."); a no-op unless a tool is attached
    NvtxRange nvtx_range(st.desc.c_str());
    if (st.kind == Step::EW) {
      EwParams p;
      to_dev(st.ew, b, &p);
      if (st.ew.finalize) {
        e = launch_finalize(p, stream);
      } else {
        EwLaunchFn sf = fn->specialize ? find_ew_spec(st.ew.sig.c_str(), st.ew.vec) : nullptr;
        e = jf ? launch_ew_fn(jf, p, st.ew.bx, st.ew.by, stream)
               : sf ? sf(p, st.ew.bx, st.ew.by, stream) : launch_ew(p, st.ew.bx, st.ew.by, stream);
      }
    } else if (st.kind == Step::GEMM) {
      const GemmStep& g = st.gemm;
      GemmParams gp;
      std::memset(&gp, 0, sizeof(gp));
      gp.M = g.M;
      gp.N = g.N;
      gp.n_seg = (int32_t)g.seg.size();
      bool aligned = true;
      for (size_t q = 0; q < g.seg.size(); ++q) {
        const GemmSeg& sg = g.seg[q];
        GemmSegParams& sp = gp.seg[q];
        const uint8_t sta = b.st[sg.a.buf], stb = b.st[sg.b.buf];
        if (sta != stb || (q > 0 && (sta == (uint8_t)SType::BF16) != (gp.bf16 != 0)))
          return fail(DLVM_ERR_RUNTIME, "dot operands with different storage types");
        gp.bf16 = sta == (uint8_t)SType::BF16;
        const size_t ea = sta == (uint8_t)SType::BF16 ? 2 : 4;
        sp.a = static_cast<const char*>(b.ptr[sg.a.buf]) + sg.a.offset * ea;
        sp.b = static_cast<const char*>(b.ptr[sg.b.buf]) + sg.b.offset * ea;
        sp.K = sg.K;
        sp.a_s0 = sg.a.strides[0];
        sp.a_s1 = sg.a.strides[1];
        sp.b_s0 = sg.b.strides[0];
        sp.b_s1 = sg.b.strides[1];
        sp.a_kmajor = sg.a_kmajor;
        sp.b_kmajor = sg.b_kmajor;
        aligned = aligned && reinterpret_cast<uintptr_t>(sp.a) % 16 == 0 && reinterpret_cast<uintptr_t>(sp.b) % 16 == 0;
      }
      gp.bm = g.bm;
      gp.bn = g.bn;
      gp.ksplit = g.ksplit;
      gp.sched = dyn && g.sched_index >= 0 ? static_cast<int*>(b.ptr[P.sched_buf]) + 2 * g.sched_index : nullptr;
      gp.hyb = hyb && g.sched_index >= 0 ? static_cast<int*>(b.ptr[P.sched_buf]) + 2 * g.sched_index : nullptr;
      gp.split_bytes = g.split_bytes;
      to_dev(g.epi, b, &gp.epi);
      gp.epi.vec = epi_vec(gp.epi);
      // L2 prefetch of row-contiguous epilogue inputs by the TMA producer warp:
      // off by default -- measured to slow the mainloop (the producer issues
      // them between its operand loads): c4 10.53 -> 10.31 ms without.
      // DLVM_GEMM_PF=1 enables it.
      static const bool epi_pf = [] {
        const char* e = std::getenv("DLVM_GEMM_PF");
        return e && e[0] == '1';
      }();
      for (int i = 1; epi_pf && i < gp.epi.prog.n_in && gp.n_pf < 4; ++i) {  // row-contiguous [M, N] epilogue inputs
        const EwDevIn& r = gp.epi.in[i];
        if (r.nchunks != 1 || r.s[1] != 1 || r.s[0] == 0) continue;
        const int es = st_bytes(r.st);
        if (reinterpret_cast<uintptr_t>(r.ptr) % 16 || (r.s[0] * es) % 16) continue;
        gp.pf_ptr[gp.n_pf] = r.ptr;
        gp.pf_row_bytes[gp.n_pf] = r.s[0] * es;
        gp.pf_esize[gp.n_pf] = es;
        ++gp.n_pf;
      }
      // K split in two with a store-only sum step after it, whose home is
      // bound as f32: zero the home and let both splits add into it
      if (g.split_red_ok && split_red_env && g.tensor_core && aligned && gp.bf16 && si + 1 < P.steps.size() &&
          P.steps[si + 1].kind == Step::EW && b.st[P.steps[si + 1].ew.stores[0].buf] == (uint8_t)SType::F32) {
        EwParams np;
        to_dev(P.steps[si + 1].ew, b, &np);
        gp.epi.out[0] = np.out[0];
        gp.epi.vec = epi_vec(gp.epi);
        gp.split_red = 1;
        e = cudaMemset2DAsync(np.out[0].ptr, (size_t)np.out[0].s[0] * 4, 0, (size_t)g.N * 4, (size_t)g.M, stream);
        if (e != cudaSuccess) return fail(DLVM_ERR_CUDA, std::string("cudaMemset2DAsync: ") + cudaGetErrorString(e));
        red_skip = (int)si + 1;
      }
      if (g.tensor_core && aligned && gp.bf16) {
        GemmLaunchFn sf = fn->specialize ? find_gemm_spec(g.epi.sig.c_str(), g.bn) : nullptr;
        e = jf ? launch_gemm_tc_fn(jf, gemm_tc_ctas(gp.M, gp.bn), gp, stream) : sf ? sf(gp, stream) : launch_gemm_tc(gp, stream);
      }
      else {
        if (g.tensor_core) return fail(DLVM_ERR_RUNTIME, "tensor-core dot operand misaligned");
        GemmLaunchFn sf = fn->specialize ? find_simt_spec(g.epi.sig.c_str(), g.bm) : nullptr;
        e = jf && gp.bf16 == (g.seg[0].a.st == SType::BF16) ? launch_gemm_simt_fn(jf, gp, stream)
            : sf ? sf(gp, stream) : launch_gemm_simt(gp, stream);
      }
    } else if (st.kind == Step::CAST) {
      const dlvm_tensor& src = param(st.cast.input);
      const bool f32 = src.dtype == DLVM_F32;
      if (st.cast.ld)
        e = launch_pack_bf16(src.data, f32, st.cast.numel / st.cast.cols, st.cast.cols, b.ptr[st.cast.dst_buf],
                             st.cast.ld, stream);
      else if (f32)
        e = launch_cast_bf16(static_cast<const float*>(src.data), b.ptr[st.cast.dst_buf], st.cast.numel, stream);
    } else if (st.kind == Step::EVENT) {
      if (events && events[st.event_index]) e = cudaEventRecord(static_cast<cudaEvent_t>(events[st.event_index]), stream);
    }
    if (e != cudaSuccess) return fail(DLVM_ERR_CUDA, std::string("CUDA error in '") + st.desc + "': " + cudaGetErrorString(e));
    if (conc && fn->step_signals[which][si] && (e = cudaEventRecord(fn->events[si], stream)) != cudaSuccess)
      return fail(DLVM_ERR_CUDA, std::string("cudaEventRecord: ") + cudaGetErrorString(e));
  }
  if (conc) {  // join: the caller's stream continues after the auxiliary one
    stream = stream_main;
    cudaError_t e = cudaEventRecord(fn->events[nsteps], fn->aux);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(stream_main, fn->events[nsteps], 0);
    if (e != cudaSuccess) return fail(DLVM_ERR_CUDA, std::string("join: ") + cudaGetErrorString(e));
    (void)aux_used;
  }
  if (!lev.empty()) {
    cudaError_t e = mark(li);
    if (e != cudaSuccess) return fail(DLVM_ERR_CUDA, std::string("cudaEventRecord: ") + cudaGetErrorString(e));
  }
  return DLVM_OK;
}

// minimum bytes a launch moves: each distinct input read once, each output written once
double step_bytes(const Plan& P, const Step& st) {
  if (st.kind == Step::CAST) return (double)st.cast.numel * 2 + (double)(st.cast.numel / st.cast.cols) * st.cast.ld * 2;
  const EwGroup& g = st.kind == Step::GEMM ? st.gemm.epi : st.ew;
  auto esz = [&](int buf, SType fallback) {
    SType t = buf >= 0 ? P.bufs[buf].st : fallback;
    return (double)st_bytes((uint8_t)t);
  };
  double b = 0;
  if (st.kind == Step::EW && st.ew.finalize) {
    // a merged finalize: input q is the [nchunks, dims[q]] partials of
    // reduction q (dims[q] its own length); store o writes dims[store_slot[o]]
    for (size_t q = 0; q < g.inputs.size(); ++q)
      b += (double)g.inputs[q].nchunks * (double)g.dims[q] * 4.0;
    for (size_t o = 0; o < g.stores.size(); ++o)
      b += (double)g.dims[g.prog.store_slot[o]] * esz(g.stores[o].buf, g.stores[o].st);
    return b;
  }
  int64_t n = 1;
  for (int d = 0; d < g.ndims; ++d) n *= g.dims[d];
  for (auto& r : g.inputs) {
    if (r.buf < 0) continue;
    int64_t cnt = r.nchunks;  // elements touched: product of dims with a nonzero stride
    for (int d = 0; d < g.ndims; ++d)
      if (r.strides[d] != 0) cnt *= g.dims[d];
    b += cnt * esz(r.buf, r.st);
  }
  for (auto& r : g.stores) b += n * esz(r.buf, r.st);
  for (auto& r : g.reduces) (void)r;
  if (st.kind == Step::GEMM) {
    const GemmStep& m = st.gemm;
    for (auto& sg : m.seg) {
      double e = m.tensor_core || P.bufs[sg.a.buf].st == SType::BF16 ? 2.0 : 4.0;
      b += (double)(m.M * sg.K + sg.K * m.N) * e;
    }
  }
  return b;
}

// Create-time specialisation (jit.h): every EW / GEMM step whose program is
// not in the ahead-of-time registry is compiled by NVRTC with the program as
// C++ types -- the same template the registry instantiates.  A failure
// leaves the step on the interpreter and is listed by print mode 8.
bool force_jit() {  // DLVM_FORCE_JIT=1: ignore the ahead-of-time registry (testing the JIT path)
  static const bool on = [] {
    const char* e = std::getenv("DLVM_FORCE_JIT");
    return e && e[0] == '1';
  }();
  return on;
}

void jit_specialise(dlvm_fn h) {
  std::vector<JitRequest> reqs;
  std::vector<std::pair<int, size_t>> where;
  for (int w = 0; w < 2; ++w) {
    if (!h->planned[w]) continue;
    const Plan& P = h->plan[w];
    h->jit_fn[w].assign(P.steps.size(), nullptr);
    const bool bf = h->opts.dot_precision == DLVM_DOT_BF16;
    for (size_t si = 0; si < P.steps.size(); ++si) {
      const Step& st = P.steps[si];
      std::string expr;
      if (st.kind == Step::EW && !st.ew.finalize && (force_jit() || !find_ew_spec(st.ew.sig.c_str(), st.ew.vec))) {
        bool row_red = false;
        for (int q = 0; q < st.ew.prog.n_reduces; ++q) row_red |= st.ew.prog.reduce_kind[q] == RED_ROW;
        const bool two_d = st.ew.ndims == 2 && st.ew.ncols == 1 && !row_red;
        expr = std::string("&dlvm::kern::") + (two_d ? "ew2d_kernel<" : "ew_kernel<") + std::to_string(st.ew.vec) +
               ", " + jit_prog_type(st.ew.sig) + ">";
      } else if (st.kind == Step::GEMM && st.gemm.tensor_core && (force_jit() || !find_gemm_spec(st.gemm.epi.sig.c_str(), st.gemm.bn))) {
        expr = "&dlvm::kern::gemm_tc_kernel<" + std::to_string(st.gemm.bn) + ", " + jit_prog_type(st.gemm.epi.sig) +
               ", " + std::to_string(gemm_tc_ctas(st.gemm.M, st.gemm.bn)) + ">";
      } else if (st.kind == Step::GEMM && !st.gemm.tensor_core && (force_jit() || !find_simt_spec(st.gemm.epi.sig.c_str(), st.gemm.bm))) {
        expr = std::string("&dlvm::kern::simt::gemm_simt_kernel<") + (bf ? "true" : "false") + ", " +
               std::to_string(st.gemm.bm) + ", " + jit_prog_type(st.gemm.epi.sig) + ">";
      }
      if (expr.empty()) continue;
      reqs.push_back(JitRequest{expr});
      where.emplace_back(w, si);
    }
  }
  jit_build(reqs);
  std::ostringstream rep;
  for (size_t i = 0; i < reqs.size(); ++i) {
    h->jit_fn[where[i].first][where[i].second] = reqs[i].function;
    rep << (where[i].first ? "grad" : "primal") << " step " << where[i].second << ": "
        << (reqs[i].function ? "specialised " : "interpreted (" + reqs[i].error.substr(0, 200) + ") ") << reqs[i].expr
        << "\n";
  }
  h->jit_report = rep.str();
}

}  // namespace

extern "C" {

dlvm_status dlvm_fn_create(const char* module_text, size_t len, const char* fn_name, const char* grad_name,
                           const dlvm_options* opts, dlvm_fn* out) {
  if (!module_text || !fn_name || !out) return fail(DLVM_ERR_USAGE, "NULL argument");
  *out = nullptr;
  dlvm_options o{};
  o.dot_precision = DLVM_DOT_F32;
  o.device = -1;
  if (opts) o = *opts;
  if (o.dot_precision != DLVM_DOT_F32 && o.dot_precision != DLVM_DOT_BF16)
    return fail(DLVM_ERR_USAGE, "unknown dot precision");
  if (o.device < -1) return fail(DLVM_ERR_USAGE, "device must be -1 (current) or a device ordinal");
  try {
    Module m = parse_module(std::string(module_text, len));
    verify_module(m);
    if (!m.find(fn_name)) return fail(DLVM_ERR_USAGE, std::string("no function @") + fn_name);
    // a gradient declaration as the primal is canonicalised first, so `grad`
    // may differentiate a gradient function (higher order)
    const Function primal = canonical_function(m, fn_name);
    const Function* src = &primal;
    Function* decl = nullptr;
    if (grad_name) {
      decl = m.find(grad_name);
      if (!decl || !decl->grad || decl->grad->source != fn_name)
        return fail(DLVM_ERR_USAGE, std::string("@") + grad_name + " is not a gradient declaration of @" + fn_name);
    } else {
      int n = 0;
      for (auto& g : m.fns)
        if (g.grad && g.grad->source == fn_name) {
          decl = &g;
          ++n;
        }
      if (n > 1) decl = nullptr;
    }
    auto* h = new (std::nothrow) dlvm_fn_s;
    if (!h) return fail(DLVM_ERR_RUNTIME, "out of host memory");
    h->opts = o;
    h->specialize = (o.flags & DLVM_NO_SPECIALIZE) == 0;
    h->primal = *src;
    if (decl) {
      h->grad = differentiate(*src, *decl->grad, decl->name);
      int nw = decl->grad->has_wrt ? (int)decl->grad->wrt.size() : src->num_args();
      h->n_grads = nw;
    }
    h->opt_primal = h->primal;
    if (h->grad) h->opt_grad = *h->grad;
    if (!(o.flags & DLVM_NO_OPT)) {
      optimize_function(h->opt_primal);
      if (h->opt_grad) optimize_function(*h->opt_grad);
    }
    for (int which = 0; which < 2; ++which) {
      if (which == 1 && !h->grad) continue;
      PlanOptions po;
      po.policy = o.dot_precision == DLVM_DOT_BF16 ? Policy::BF16 : Policy::F32;
      po.no_fusion = (o.flags & DLVM_NO_FUSION) != 0;
      po.specialize = (o.flags & DLVM_NO_SPECIALIZE) == 0;
      po.n_grads = which ? h->n_grads : 0;
      try {
        h->plan[which] = make_plan(which ? *h->opt_grad : h->opt_primal, po);
        h->planned[which] = true;
        h->out_read[which] = outputs_read(h->plan[which]);
        plan_streams(h, which);
      } catch (const Error& e) {
        h->plan_error[which] = e.what();
        if (!(o.flags & DLVM_PLAN_ONLY)) {
          dlvm_status st = from_error(e);
          delete h;
          return st;
        }
      }
    }
    if (!(o.flags & (DLVM_PLAN_ONLY | DLVM_NO_SPECIALIZE | DLVM_NO_JIT)) && jit_available()) {
      // create-time kernels are loaded into the context of the run device
      DeviceGuard dg;
      if (o.device >= 0 && dg.set(o.device) != cudaSuccess) {
        delete h;
        return fail(DLVM_ERR_CUDA, "cudaSetDevice failed for dlvm_options.device");
      }
      jit_specialise(h);
    }
    *out = h;
    return DLVM_OK;
  } catch (const Error& e) {
    return from_error(e);
  } catch (const std::exception& e) {
    return fail(DLVM_ERR_RUNTIME, std::string("internal error: ") + e.what());
  } catch (...) {
    return fail(DLVM_ERR_RUNTIME, "internal error");
  }
}

dlvm_status dlvm_fn_signature(dlvm_fn fn, int which, int* n_in, dlvm_tensor* in_types, int* n_out,
                              dlvm_tensor* out_types) {
  if (!fn || !n_in || !n_out) return fail(DLVM_ERR_USAGE, "NULL argument");
  if (which == 1 && !fn->grad) return fail(DLVM_ERR_USAGE, "handle has no gradient function");
  if (which != 0 && which != 1) return fail(DLVM_ERR_USAGE, "which must be 0 or 1");
  const Function& f = which ? *fn->grad : fn->primal;
  int ci = *n_in, co = *n_out;
  *n_in = (int)f.params.size();
  *n_out = (int)f.results.size();
  for (int i = 0; i < *n_in && i < ci && in_types; ++i) fill_sig(f.params[i], &in_types[i]);
  for (int i = 0; i < *n_out && i < co && out_types; ++i) fill_sig(f.results[i], &out_types[i]);
  return DLVM_OK;
}

dlvm_status dlvm_fn_print(dlvm_fn fn, int which, char* buf, size_t cap, size_t* needed) {
  if (!fn) return fail(DLVM_ERR_USAGE, "NULL handle");
  std::string s;
  try {
    switch (which) {
      case 0: s = print_function(fn->primal); break;
      case 1:
        if (!fn->grad) return fail(DLVM_ERR_USAGE, "handle has no gradient function");
        s = print_function(*fn->grad);
        break;
      case 2:
      case 3: {
        int w = which - 2;
        if (w == 1 && !fn->grad) return fail(DLVM_ERR_USAGE, "handle has no gradient function");
        s = fn->planned[w] ? fn->plan[w].str() : "unsupported: " + fn->plan_error[w] + "\n";
        break;
      }
      case 4:
      case 5: {
        int w = which - 4;
        if (w == 1 && !fn->grad) return fail(DLVM_ERR_USAGE, "handle has no gradient function");
        if (!fn->planned[w]) return fail(DLVM_ERR_UNSUPPORTED, fn->plan_error[w]);
        for (const Step& st : fn->plan[w].steps) {
          if (st.kind == Step::EW && !st.ew.finalize)  // finalize has a fixed kernel of its own
            s += "EW " + std::to_string(st.ew.vec) + " " + st.ew.sig + "\n";
          else if (st.kind == Step::GEMM && st.gemm.tensor_core)
            s += "GEMM " + std::to_string(st.gemm.bn) + " " + st.gemm.epi.sig + "\n";
          else if (st.kind == Step::GEMM)
            s += "SIMT " + std::to_string(st.gemm.bm) + " " + st.gemm.epi.sig + "\n";
        }
        break;
      }
      case 6:
        s = print_function(fn->opt_primal);
        break;
      case 7:
        if (!fn->opt_grad) return fail(DLVM_ERR_USAGE, "handle has no gradient function");
        s = print_function(*fn->opt_grad);
        break;
      case 8:
        s = fn->jit_report;
        break;
      case 9:
      case 10: {
        int w = which - 9;
        if (w == 1 && !fn->grad) return fail(DLVM_ERR_USAGE, "handle has no gradient function");
        s = fn->planned[w] ? fn->plan[w].detail() : "unsupported: " + fn->plan_error[w] + "\n";
        break;
      }
      case 11:
      case 12: {  // two-stream schedule of the primal (11) / gradient (12)
        int w = which - 11;
        if (w == 1 && !fn->grad) return fail(DLVM_ERR_USAGE, "handle has no gradient function");
        if (!fn->planned[w]) return fail(DLVM_ERR_UNSUPPORTED, fn->plan_error[w]);
        const Plan& P = fn->plan[w];
        s = std::string("streams: ") + (fn->concurrent[w] ? "two" : "one") + "\n";
        for (size_t i = 0; i < P.steps.size(); ++i) {
          s += "  [" + std::to_string(i) + "] " + (fn->step_stream[w][i] ? "aux " : "main") + " ";
          for (int k : fn->step_waits[w][i]) s += "wait[" + std::to_string(k) + "] ";
          s += P.steps[i].desc.substr(0, 60) + "\n";
        }
        break;
      }
      default:
        return fail(DLVM_ERR_USAGE, "which must be 0..12");
    }
  } catch (const std::exception& e) {
    return fail(DLVM_ERR_RUNTIME, e.what());
  }
  if (needed) *needed = s.size() + 1;
  if (buf && cap) {
    size_t n = std::min(cap - 1, s.size());
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  return DLVM_OK;
}

dlvm_status dlvm_fn_workspace_bytes(dlvm_fn fn, int which, size_t* bytes) {
  if (!fn || !bytes) return fail(DLVM_ERR_USAGE, "NULL argument");
  if (which != 0 && which != 1) return fail(DLVM_ERR_USAGE, "which must be 0 or 1");
  if (which == 1 && !fn->grad) return fail(DLVM_ERR_USAGE, "handle has no gradient function");
  if (!fn->planned[which]) return fail(DLVM_ERR_UNSUPPORTED, fn->plan_error[which]);
  *bytes = fn->plan[which].workspace_bytes;
  return DLVM_OK;
}

dlvm_status dlvm_fn_num_launches(dlvm_fn fn, int which, int* launches) {
  if (!fn || !launches) return fail(DLVM_ERR_USAGE, "NULL argument");
  if (which != 0 && which != 1) return fail(DLVM_ERR_USAGE, "which must be 0 or 1");
  if (which == 1 && !fn->grad) return fail(DLVM_ERR_USAGE, "handle has no gradient function");
  if (!fn->planned[which]) return fail(DLVM_ERR_UNSUPPORTED, fn->plan_error[which]);
  *launches = fn->plan[which].launches();
  return DLVM_OK;
}

dlvm_status dlvm_fn_run(dlvm_fn fn, const dlvm_tensor* in, int n_in, dlvm_tensor* out, int n_out, void* workspace,
                        void* cuda_stream) {
  try {
    return execute(fn, 0, in, n_in, nullptr, out, n_out, workspace, cuda_stream, nullptr);
  } catch (const std::exception& e) {
    return fail(DLVM_ERR_RUNTIME, e.what());
  }
}

dlvm_status dlvm_grad_run(dlvm_fn fn, const dlvm_tensor* in, int n_in, const dlvm_tensor* seed, dlvm_tensor* out,
                          int n_out, void* workspace, void* cuda_stream, void* const* grad_ready_events) {
  if (fn && !fn->grad) return fail(DLVM_ERR_USAGE, "handle has no gradient function");
  try {
    return execute(fn, 1, in, n_in, seed, out, n_out, workspace, cuda_stream, grad_ready_events);
  } catch (const std::exception& e) {
    return fail(DLVM_ERR_RUNTIME, e.what());
  }
}

dlvm_status dlvm_fn_launch_events(dlvm_fn fn, int which, void* const* events, int n_events) {
  if (!fn || (which != 0 && which != 1)) return fail(DLVM_ERR_USAGE, "bad handle or which");
  if (which == 1 && !fn->grad) return fail(DLVM_ERR_USAGE, "handle has no gradient function");
  if (!fn->planned[which]) return fail(DLVM_ERR_UNSUPPORTED, fn->plan_error[which]);
  if (!events || n_events == 0) {
    fn->launch_events[which].clear();
    return DLVM_OK;
  }
  if (n_events != fn->plan[which].launches() + 1) return fail(DLVM_ERR_USAGE, "n_events must be launches + 1");
  fn->launch_events[which].assign(events, events + n_events);
  return DLVM_OK;
}

dlvm_status dlvm_fn_launch_info(dlvm_fn fn, int which, int i, char* buf, size_t cap, double* flops, double* bytes) {
  if (!fn || (which != 0 && which != 1)) return fail(DLVM_ERR_USAGE, "bad handle or which");
  if (which == 1 && !fn->grad) return fail(DLVM_ERR_USAGE, "handle has no gradient function");
  if (!fn->planned[which]) return fail(DLVM_ERR_UNSUPPORTED, fn->plan_error[which]);
  const Plan& P = fn->plan[which];
  int li = 0;
  for (const Step& st : P.steps) {
    if (!st.counted_launch()) continue;
    if (li++ != i) continue;
    if (buf && cap) {
      size_t n = std::min(cap - 1, st.desc.size());
      std::memcpy(buf, st.desc.data(), n);
      buf[n] = 0;
    }
    if (flops) flops[0] = st.kind == Step::GEMM ? 2.0 * st.gemm.M * st.gemm.N * st.gemm.K : 0.0;
    if (bytes) bytes[0] = step_bytes(P, st);
    return DLVM_OK;
  }
  return fail(DLVM_ERR_USAGE, "launch index out of range");
}

const char* dlvm_last_error(void) { return g_last_error.c_str(); }

void dlvm_fn_destroy(dlvm_fn fn) { delete fn; }

const char* dlvm_version(void) { return "dlvm-b200 0.1 sm_100a"; }

}  // extern "C"

// tcgen05 GEMM entry points (kernel template in gemm_tc.cuh): the generic
// instantiation whose epilogue interprets the planner's program, and the
// lookup of compile-time epilogue specialisations (gemm_tc_spec*.cu).
#include <cstring>

#include "gemm_tc.cuh"

namespace dlvm {

const GemmSpecEntry* gemm_spec_table_0();
const GemmSpecEntry* gemm_spec_table_1();
const GemmSpecEntry* gemm_spec_table_2();
const GemmSpecEntry* gemm_spec_table_3();

bool gemm_tc_available() { return get_encode() != nullptr; }

cudaError_t launch_gemm_tc(const GemmParams& p, cudaStream_t stream) {
  const EwProgram& e = p.epi.prog;
  const int cw = epi_chunk_width(e.n_in + e.n_lits + e.n_ins);
  if (p.bn == 256) {
    if (cw == 16) return launch_prog<256, VmEpi<16>>(p, stream);
    if (cw == 8) return launch_prog<256, VmEpi<8>>(p, stream);
    return launch_prog<256, VmEpi<4>>(p, stream);
  }
  if (cw == 16) return launch_prog<128, VmEpi<16>>(p, stream);
  if (cw == 8) return launch_prog<128, VmEpi<8>>(p, stream);
  return launch_prog<128, VmEpi<4>>(p, stream);
}

bool gemm_hybrid_enabled() { return mc_mode() == 1; }

int gemm_tc_ctas(int64_t M, int bn) {
  GemmParams p;
  std::memset(&p, 0, sizeof(p));
  p.M = M;
  p.bn = bn;
  return use_cta_pair(p) ? 2 : 1;
}

cudaError_t launch_gemm_tc_fn(void* fn, int ctas, const GemmParams& p, cudaStream_t stream) {
  TcParams tp;
  if (!make_params(p, &tp, ctas, true)) return cudaErrorInvalidValue;  // NVRTC kernels run compile-time programs
  const int smem = launch_smem(tp, p.bn, ctas);
  int cluster = 1, grid = 1;
  grid_of(tp, ctas, &cluster, &grid);
  LaunchCfg L(dim3((unsigned)grid, 1, 1), dim3(NUM_THREADS, 1, 1), smem, stream, (unsigned)cluster, 1);
  void* args[] = {&tp};
  return launch_jit(fn, L, args);
}

GemmLaunchFn find_gemm_spec(const char* sig, int bn) {
  const GemmSpecEntry* tabs[4] = {gemm_spec_table_0(), gemm_spec_table_1(), gemm_spec_table_2(),
                                  gemm_spec_table_3()};
  for (auto* t : tabs)
    for (const GemmSpecEntry* e = t; e->sig; ++e)
      if (e->fn && e->bn == bn && std::strcmp(e->sig, sig) == 0) return e->fn;
  return nullptr;
}

int num_gemm_specs() {
  int n = 0;
  const GemmSpecEntry* tabs[4] = {gemm_spec_table_0(), gemm_spec_table_1(), gemm_spec_table_2(),
                                  gemm_spec_table_3()};
  for (auto* t : tabs)
    for (const GemmSpecEntry* e = t; e->sig; ++e) n += e->fn != nullptr;
  return n;
}

}  // namespace dlvm

#ifdef DLVM_GEMM_TRACE
// Trace builds only (not part of dlvm.h): tcgen05 GEMM launches k = 0, 1, ...
// after this call write their phase stamps to slice k % slots of `dev`
// ([slots][148][32] u64, caller-owned device memory); NULL stops tracing.
// Used by tools/gemm_trace.py.
namespace dlvm {
namespace kern {
unsigned long long* g_gemm_trace_ptr = nullptr;
int g_gemm_trace_slots = 1, g_gemm_trace_next = 0;
}  // namespace kern
}  // namespace dlvm
extern "C" void dlvm_debug_gemm_trace(void* dev, int slots) {
  dlvm::kern::g_gemm_trace_ptr = static_cast<unsigned long long*>(dev);
  dlvm::kern::g_gemm_trace_slots = slots > 0 ? slots : 1;
  dlvm::kern::g_gemm_trace_next = 0;
}
#endif

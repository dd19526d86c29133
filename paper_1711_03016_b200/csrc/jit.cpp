// Create-time kernel specialisation with NVRTC (see jit.h).
#include "jit.h"

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nvrtc.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <mutex>
#include <sstream>
#include <thread>

namespace dlvm {

namespace {

namespace fs = std::filesystem;

struct Nvrtc {
  void* h = nullptr;
  decltype(&nvrtcCreateProgram) create = nullptr;
  decltype(&nvrtcAddNameExpression) add_name = nullptr;
  decltype(&nvrtcCompileProgram) compile = nullptr;
  decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
  decltype(&nvrtcGetProgramLog) get_log = nullptr;
  decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
  decltype(&nvrtcGetCUBIN) get_cubin = nullptr;
  decltype(&nvrtcGetLoweredName) lowered = nullptr;
  decltype(&nvrtcDestroyProgram) destroy = nullptr;
  bool ok = false;
};

const Nvrtc& nvrtc() {
  static Nvrtc n;
  static std::once_flag once;
  std::call_once(once, [] {
    for (const char* lib : {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12"}) {
      n.h = dlopen(lib, RTLD_NOW | RTLD_LOCAL);
      if (n.h) break;
    }
    if (!n.h) return;
#define DLVM_SYM(field, name) n.field = reinterpret_cast<decltype(n.field)>(dlsym(n.h, #name))
    DLVM_SYM(create, nvrtcCreateProgram);
    DLVM_SYM(add_name, nvrtcAddNameExpression);
    DLVM_SYM(compile, nvrtcCompileProgram);
    DLVM_SYM(log_size, nvrtcGetProgramLogSize);
    DLVM_SYM(get_log, nvrtcGetProgramLog);
    DLVM_SYM(cubin_size, nvrtcGetCUBINSize);
    DLVM_SYM(get_cubin, nvrtcGetCUBIN);
    DLVM_SYM(lowered, nvrtcGetLoweredName);
    DLVM_SYM(destroy, nvrtcDestroyProgram);
#undef DLVM_SYM
    n.ok = n.create && n.add_name && n.compile && n.log_size && n.get_log && n.cubin_size && n.get_cubin &&
           n.lowered && n.destroy;
  });
  return n;
}

struct Driver {
  PFN_cuModuleLoadData_v2000 load = nullptr;
  PFN_cuModuleGetFunction_v2000 get_function = nullptr;
  bool ok = false;
};

const Driver& driver() {
  static Driver d;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuModuleLoadData", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      d.load = reinterpret_cast<PFN_cuModuleLoadData_v2000>(p);
    if (cudaGetDriverEntryPoint("cuModuleGetFunction", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      d.get_function = reinterpret_cast<PFN_cuModuleGetFunction_v2000>(p);
    d.ok = d.load && d.get_function;
  });
  return d;
}

// directory of the kernel headers: $DLVM_KERNEL_SRC, else csrc/kernels next
// to this shared library
std::string kernel_dir() {
  if (const char* e = std::getenv("DLVM_KERNEL_SRC")) return e;
  Dl_info info;
  if (dladdr(reinterpret_cast<void*>(&jit_available), &info) && info.dli_fname) {
    fs::path so(info.dli_fname);
    return (so.parent_path() / "csrc" / "kernels").string();
  }
  return "";
}

std::string cuda_include() {
  if (const char* e = std::getenv("CUDA_HOME")) return std::string(e) + "/include";
  return "/usr/local/cuda/include";
}

uint64_t fnv(uint64_t h, const std::string& s) {
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ull;
  }
  return h;
}

// hash of every kernel header: a changed template invalidates cached cubins
uint64_t source_hash() {
  static uint64_t h = 0;
  static std::once_flag once;
  std::call_once(once, [] {
    uint64_t x = 1469598103934665603ull;
    std::vector<fs::path> files;
    std::error_code ec;
    for (auto& e : fs::directory_iterator(kernel_dir(), ec)) {
      const auto ext = e.path().extension().string();
      if (ext == ".cuh" || ext == ".h" || ext == ".inc") files.push_back(e.path());
    }
    std::sort(files.begin(), files.end());
    for (auto& f : files) {
      std::ifstream in(f, std::ios::binary);
      std::stringstream ss;
      ss << in.rdbuf();
      x = fnv(fnv(x, f.filename().string()), ss.str());
    }
    h = x;
  });
  return h;
}

std::string cache_dir() {
  if (const char* e = std::getenv("DLVM_JIT_CACHE")) return e;
  const char* home = std::getenv("HOME");
  return std::string(home ? home : "/tmp") + "/.cache/dlvm-jit";
}

const char* kSource =
    "#include \"gemm_tc_kernel.cuh\"\n"
    "#include \"gemm_simt_kernel.cuh\"\n";

std::vector<std::string> options() {
  std::vector<std::string> o = {"--gpu-architecture=sm_100a", "-std=c++17", "-default-device", "-lineinfo",
                                "-I" + kernel_dir(), "-I" + cuda_include()};
  // a build variant's kernel-layout defines apply to create-time kernels too
  // (they are part of the cache key below)
#ifdef DLVM_GEMM_TRACE
  o.push_back("-DDLVM_GEMM_TRACE");
#endif
#ifdef DLVM_GEMM_STAGES_PAIR
  o.push_back("-DDLVM_GEMM_STAGES_PAIR=" + std::to_string(DLVM_GEMM_STAGES_PAIR));
#endif
#ifdef DLVM_EW_RPI
  o.push_back("-DDLVM_EW_RPI=" + std::to_string(DLVM_EW_RPI));
#endif
  return o;
}

// NVRTC compile of one instantiation -> (lowered name, cubin)
bool compile_one(const std::string& expr, std::string* lowered, std::string* cubin, std::string* err) {
  const Nvrtc& n = nvrtc();
  nvrtcProgram prog;
  if (n.create(&prog, kSource, "dlvm_jit.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
    *err = "nvrtcCreateProgram failed";
    return false;
  }
  n.add_name(prog, expr.c_str());
  std::vector<std::string> o = options();
  std::vector<const char*> ov;
  for (auto& s : o) ov.push_back(s.c_str());
  const nvrtcResult r = n.compile(prog, (int)ov.size(), ov.data());
  if (r != NVRTC_SUCCESS) {
    size_t ls = 0;
    n.log_size(prog, &ls);
    std::string log(ls, '\0');
    n.get_log(prog, log.data());
    *err = "NVRTC: " + log.substr(0, 4000);
    n.destroy(&prog);
    return false;
  }
  const char* low = nullptr;
  n.lowered(prog, expr.c_str(), &low);
  *lowered = low ? low : "";
  size_t cs = 0;
  n.cubin_size(prog, &cs);
  cubin->assign(cs, '\0');
  n.get_cubin(prog, cubin->data());
  n.destroy(&prog);
  return !lowered->empty() && cs > 0;
}

bool cached_compile(const std::string& expr, std::string* lowered, std::string* cubin, std::string* err) {
  std::string key;
  for (auto& o : options()) key += o + "\n";
  char name[64];
  std::snprintf(name, sizeof(name), "%016llx.cubin",
                (unsigned long long)fnv(fnv(source_hash(), key), expr));
  const fs::path path = fs::path(cache_dir()) / name;
  {
    std::ifstream in(path, std::ios::binary);
    if (in) {
      std::getline(in, *lowered);
      std::stringstream ss;
      ss << in.rdbuf();
      *cubin = ss.str();
      if (!lowered->empty() && !cubin->empty()) return true;
    }
  }
  if (!compile_one(expr, lowered, cubin, err)) return false;
  std::error_code ec;
  fs::create_directories(path.parent_path(), ec);
  const fs::path tmp = path.string() + ".tmp" + std::to_string(::getpid()) + "_" +
                       std::to_string(std::hash<std::thread::id>{}(std::this_thread::get_id()));
  {
    std::ofstream out(tmp, std::ios::binary);
    out << *lowered << "\n";
    out.write(cubin->data(), (std::streamsize)cubin->size());
  }
  fs::rename(tmp, path, ec);  // best effort: a read-only cache still works
  if (ec) fs::remove(tmp, ec);
  return true;
}

}  // namespace

bool jit_available() {
  const char* e = std::getenv("DLVM_JIT");
  if (e && e[0] == '0') return false;
  return nvrtc().ok && !kernel_dir().empty();
}

std::string jit_prog_type(const std::string& sig) {
  // "i<nin>l<nlit>|op,a,b,c;...|s<slot>,..|r<slot>:<kind>,.." (plan.cpp program_signature)
  std::vector<std::string> parts;
  std::stringstream ss(sig);
  std::string item;
  while (std::getline(ss, item, '|')) parts.push_back(item);
  while (parts.size() < 4) parts.push_back("");
  const size_t lpos = parts[0].find('l');
  const int nin = std::atoi(parts[0].substr(1, lpos - 1).c_str());
  const int nlit = std::atoi(parts[0].substr(lpos + 1).c_str());
  std::string out = "dlvm::spec::Prog<" + std::to_string(nin) + ", " + std::to_string(nlit) + ", dlvm::spec::St<";
  out += parts[2].size() > 1 ? parts[2].substr(1) : "";
  out += ">, dlvm::spec::Rd<";
  std::string rd = parts[3].size() > 1 ? parts[3].substr(1) : "";
  std::replace(rd.begin(), rd.end(), ':', ',');
  out += rd + ">";
  int k = 0;
  std::stringstream is(parts[1]);
  while (std::getline(is, item, ';')) {
    if (item.empty()) continue;
    int op, a, b, c;
    if (std::sscanf(item.c_str(), "%d,%d,%d,%d", &op, &a, &b, &c) != 4) continue;
    out += ", dlvm::spec::Ins<" + std::to_string(op) + ", " + std::to_string(nin + nlit + k) + ", " +
           std::to_string(a) + ", " + std::to_string(b) + ", " + std::to_string(c) + ">";
    ++k;
  }
  return out + ">";
}

bool jit_build(std::vector<JitRequest>& reqs) {
  if (reqs.empty()) return true;
  if (!jit_available() || !driver().ok) {
    for (auto& r : reqs) r.error = "JIT unavailable";
    return false;
  }
  std::vector<std::string> lowered(reqs.size()), cubin(reqs.size());
  std::vector<char> ok(reqs.size(), 0);
  std::atomic<size_t> next{0};
  const unsigned nt = std::max(1u, std::min<unsigned>((unsigned)reqs.size(), std::min(8u, std::thread::hardware_concurrency())));
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < nt; ++t)
    pool.emplace_back([&] {
      for (size_t i; (i = next++) < reqs.size();)
        ok[i] = cached_compile(reqs[i].expr, &lowered[i], &cubin[i], &reqs[i].error) ? 1 : 0;
    });
  for (auto& t : pool) t.join();
  cudaFree(nullptr);  // make the device's primary context current for the module loads
  bool all = true;
  for (size_t i = 0; i < reqs.size(); ++i) {
    if (!ok[i]) {
      all = false;
      continue;
    }
    CUmodule mod;
    CUfunction fn;
    if (driver().load(&mod, cubin[i].data()) != CUDA_SUCCESS ||
        driver().get_function(&fn, mod, lowered[i].c_str()) != CUDA_SUCCESS) {
      reqs[i].error = "loading the JIT cubin failed";
      all = false;
      continue;
    }
    reqs[i].function = fn;  // modules stay loaded for the process
  }
  return all;
}

}  // namespace dlvm

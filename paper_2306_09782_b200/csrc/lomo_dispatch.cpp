// lomo_dispatch.cpp -- the hook-side launcher of K1/K2 in C++ (a torch
// extension module, _lomo_dispatch).
//
// The autograd hook (lomo.py, tape.py:387-405 boundary) hands each complete
// gradient to the dispatcher, which launches K1 (update) or K2 (probe) through
// the C-ABI (include/lomo_b200.h) on the hook's CUDA stream, or parks tiny
// tensors (the RMSNorm scales) for one multi-tensor launch per 64 at the end
// of the pass.  The Python form of the same logic (dispatch.HookDispatcher)
// spends ~6-20 us of interpreter and ctypes argument conversion per launch;
// here a launch costs one pybind call plus the CUDA launch itself.
//
// The module holds no compute of its own: every kernel is the C-ABI's.
#include <torch/extension.h>

#include <cstdint>
#include <map>
#include <utility>
#include <vector>

#include "lomo_b200.h"

namespace {

int dtype_code(const at::Tensor& t) {
  switch (t.scalar_type()) {
    case at::kFloat: return LOMO_F32;
    case at::kHalf: return LOMO_F16;
    case at::kBFloat16: return LOMO_BF16;
    case at::kDouble: return LOMO_F64;
    default: TORCH_CHECK(false, "lomo: unsupported dtype ", t.scalar_type());
  }
  return -1;
}

void check(int rc, const char* what) {
  TORCH_CHECK(rc == 0, "lomo: ", what, " failed with status ", rc);
}

class Dispatcher {
 public:
  Dispatcher(int64_t state_ptr, int math, int64_t small_numel)
      : state_(reinterpret_cast<void*>(state_ptr)), math_(math), small_(small_numel) {}

  // chain: consecutive K1 launches of this dispatcher on one stream are
  // declared independent (LOMO_CHAINED, dispatch.HookDispatcher.configure)
  void configure(double lr, double clip, double wd, int64_t flags, bool chain) {
    lr_ = lr;
    clip_ = clip;
    wd_ = wd;
    flags_ = (unsigned)flags;
    chain_ = chain;
    chain_kind_ = 0;
    chain_stream_ = nullptr;
  }

  // K1 for one (parameter, gradient) pair, or park it when tiny.
  void update(const at::Tensor& p, const at::Tensor& g, int64_t stream_ptr) {
    cur_ = reinterpret_cast<void*>(stream_ptr);
    const int64_t n = p.numel();
    const int dt = dtype_code(p);
    if (n <= small_) {
      auto& lst = upd_[dt];
      lst.emplace_back(p, g);
      if (lst.size() == 64) flush_upd(dt);
      return;
    }
    check(lomo_fused_update(p.data_ptr(), g.data_ptr(), n, dt, math_, lr_, clip_, wd_,
                            flags_ | chained('u'), state_, stream()),
          "lomo_fused_update");
    mark('u');
    ++launches_;
  }

  // K2 for one gradient into norm slot `slot`, or park it when tiny.
  void probe(const at::Tensor& g, int64_t slot, int64_t stream_ptr) {
    cur_ = reinterpret_cast<void*>(stream_ptr);
    const int64_t n = g.numel();
    const int dt = dtype_code(g);
    if (n <= small_) {
      auto& lst = prb_[dt];
      lst.emplace_back(g, (int)slot);
      if (lst.size() == 64) flush_prb(dt);
      return;
    }
    check(lomo_probe(g.data_ptr(), n, dt, (int)slot, flags_ | chained('p'), state_, stream()),
          "lomo_probe");
    mark('p');
    ++launches_;
  }

  void flush(int64_t stream_ptr) {
    cur_ = reinterpret_cast<void*>(stream_ptr);
    std::vector<int> ks;
    for (auto& kv : upd_) ks.push_back(kv.first);
    for (int dt : ks) flush_upd(dt);
    ks.clear();
    for (auto& kv : prb_) ks.push_back(kv.first);
    for (int dt : ks) flush_prb(dt);
  }

  int64_t pending() const {
    int64_t k = 0;
    for (auto& kv : upd_) k += (int64_t)kv.second.size();
    for (auto& kv : prb_) k += (int64_t)kv.second.size();
    return k;
  }

  int64_t launches() const { return launches_; }
  double lr() const { return lr_; }
  double clip() const { return clip_; }
  double wd() const { return wd_; }
  int64_t flags() const { return flags_; }

 private:
  // the raw cudaStream_t the caller passed (the hook's stream)
  void* stream() const { return cur_; }

  // LOMO_CHAINED when this dispatcher's previous launch on this stream was of
  // the same family ('u': K1 / K1 multi, 'p': K2 / K2 multi)
  unsigned chained(char kind) const {
    return (chain_ && chain_kind_ == kind && chain_stream_ == cur_) ? LOMO_CHAINED : 0u;
  }
  void mark(char kind) {
    chain_kind_ = kind;
    chain_stream_ = cur_;
  }

  void flush_upd(int dt) {
    auto it = upd_.find(dt);
    if (it == upd_.end() || it->second.empty()) return;
    auto& lst = it->second;
    const int k = (int)lst.size();
    std::vector<void*> ps(k);
    std::vector<const void*> gs(k);
    std::vector<int64_t> ns(k);
    for (int i = 0; i < k; ++i) {
      ps[i] = lst[i].first.data_ptr();
      gs[i] = lst[i].second.data_ptr();
      ns[i] = lst[i].first.numel();
    }
    check(lomo_fused_update_multi(ps.data(), gs.data(), ns.data(), k, dt, math_, lr_, clip_, wd_,
                                  flags_, state_, stream()),
          "lomo_fused_update_multi");
    mark('u');  // a K1 multi on other tensors may precede a chained K1
    launches_ += (k + 63) / 64;
    lst.clear();  // released after the launch: stream-ordered reuse by the allocator
  }

  void flush_prb(int dt) {
    auto it = prb_.find(dt);
    if (it == prb_.end() || it->second.empty()) return;
    auto& lst = it->second;
    const int k = (int)lst.size();
    std::vector<const void*> gs(k);
    std::vector<int64_t> ns(k);
    std::vector<int> ss(k);
    for (int i = 0; i < k; ++i) {
      gs[i] = lst[i].first.data_ptr();
      ns[i] = lst[i].first.numel();
      ss[i] = lst[i].second;
    }
    check(lomo_probe_multi(gs.data(), ns.data(), ss.data(), k, dt, flags_, state_, stream()),
          "lomo_probe_multi");
    mark('p');
    launches_ += (k + 63) / 64;
    lst.clear();
  }

  void* state_;
  void* cur_ = nullptr;
  int math_;
  int64_t small_;
  double lr_ = 0.0, clip_ = 0.0, wd_ = 0.0;
  unsigned flags_ = 0;
  bool chain_ = false;
  char chain_kind_ = 0;           // family and stream of the last launch (chain mode)
  void* chain_stream_ = nullptr;
  int64_t launches_ = 0;
  std::map<int, std::vector<std::pair<at::Tensor, at::Tensor>>> upd_;
  std::map<int, std::vector<std::pair<at::Tensor, int>>> prb_;
};

}  // namespace

PYBIND11_MODULE(TORCH_EXTENSION_NAME, m) {
  m.doc() = "C++ hook dispatcher for the LOMO C-ABI (K1/K2 launches)";
  pybind11::class_<Dispatcher>(m, "Dispatcher")
      .def(pybind11::init<int64_t, int, int64_t>())
      .def("configure", &Dispatcher::configure, pybind11::arg("lr"), pybind11::arg("clip"),
           pybind11::arg("wd"), pybind11::arg("flags"), pybind11::arg("chain") = false)
      .def("update", &Dispatcher::update)
      .def("probe", &Dispatcher::probe)
      .def("flush", &Dispatcher::flush)
      .def("pending", &Dispatcher::pending)
      .def_property_readonly("launches", &Dispatcher::launches)
      .def_property_readonly("lr", &Dispatcher::lr)
      .def_property_readonly("clip", &Dispatcher::clip)
      .def_property_readonly("wd", &Dispatcher::wd)
      .def_property_readonly("flags", &Dispatcher::flags);
  m.def("abi_version", []() { return lomo_abi_version(); });
}

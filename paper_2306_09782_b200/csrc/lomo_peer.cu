// lomo_peer.cu -- peer-memory transport for K4 (sharded mode, one process per
// GPU), behind include/lomo_b200.h.
//
// K4 (lomo_fused_rs_update / lomo_fused_mc_update) reduces a bucket's
// gradients over the ranks' own buffers instead of an NCCL reduce-scatter
// (SURVEY 8e, 8f(1)).  That needs (a) the ranks' bucket buffers mapped into
// every rank's address space and (b) a device-side barrier that orders "every
// rank finished writing the bucket" before the reads, and "every rank finished
// reading" before a buffer is refilled.  The reference has no distributed code
// (SPEC.md:454); what K4 fuses is probe_hook (stabilize.py:193-200) and the
// update (optim.py:52-54) applied to the reduced gradient.
//
//  * CUDA IPC: one cudaMalloc per rank (buffers + signal area), its handle
//    exchanged by the host, opened by every peer (lazy peer access).  Works
//    across NVLink peers and between two processes sharing one GPU.
//  * NVLS multicast (driver API): rank 0 creates the multicast object, the
//    others import it through a POSIX fd (pidfd_getfd), each binds its own
//    physical memory; K4 then reads the multicast address with
//    multimem.ld_reduce and the barrier is a multimem.red on a counter.
//
// Barriers never hang the GPU: a wait longer than the caller's timeout sets
// an error flag and returns.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <new>

#include "lomo_b200.h"

namespace lomo_peer {

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Thread t < world: signal rank t (write `epoch` into slot [channel][rank] of
// t's signal area), then wait until rank t's signal in this rank's area
// ([channel][t]) reaches `epoch`.  The kernel runs after every earlier kernel
// of the stream completed (no PDL on this launch); the system-scope fence
// then the release store publish those kernels' writes to the peers.
//
// `epochs` (non-null, the *_dev entry points): the epoch is this rank's
// device counter for the channel plus one, written back at the end -- every
// rank issues the same barrier sequence, so the counters agree, and a CUDA
// graph replaying the barrier advances them (a host epoch would be frozen
// into the graph).
__global__ void k_peer_barrier(uint64_t* const* sig, int world, int rank, int channel,
                               uint64_t epoch, int64_t timeout_ns, int* err, uint64_t* epochs) {
  const int t = threadIdx.x;
  if (epochs != nullptr) epoch = epochs[channel] + 1;
  if (t < world) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    st_release_sys(sig[t] + channel * LOMO_PEER_MAX + rank, epoch);
    const uint64_t* mine = sig[rank] + channel * LOMO_PEER_MAX + t;
    const uint64_t t0 = globaltimer();
    while (ld_acquire_sys(mine) < epoch) {
      if ((int64_t)(globaltimer() - t0) > timeout_ns) {
        atomicExch(err, 2);
        break;
      }
      __nanosleep(128);
    }
  }
  __syncthreads();
  if (epochs != nullptr && t == 0) epochs[channel] = epoch;
}

// NVLS barrier: one multimem.red.add per rank on the channel's counter -- the
// switch applies it to every rank's copy -- then wait for this GPU's copy to
// reach epoch * world.
__global__ void k_mc_barrier(uint64_t* mc, const uint64_t* uc, int world, int channel,
                             uint64_t epoch, int64_t timeout_ns, int* err, uint64_t* epochs) {
  if (threadIdx.x != 0) return;
  if (epochs != nullptr) epoch = epochs[channel] + 1;
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  asm volatile("multimem.red.release.sys.global.add.u64 [%0], %1;" ::"l"(mc + channel),
               "l"((uint64_t)1)
               : "memory");
  const uint64_t want = epoch * (uint64_t)world;
  const uint64_t t0 = globaltimer();
  while (ld_acquire_sys(uc + channel) < want) {
    if ((int64_t)(globaltimer() - t0) > timeout_ns) {
      atomicExch(err, 2);
      break;
    }
    __nanosleep(128);
  }
  if (epochs != nullptr) epochs[channel] = epoch;
}

// ---------------------------------------------------------------- multicast
struct McObj {
  CUmemGenericAllocationHandle mc = 0;
  CUmemGenericAllocationHandle mem = 0;
  CUdeviceptr uc_ptr = 0, mc_ptr = 0;
  size_t size = 0;
  int fd = -1;
  bool have_mc = false, have_mem = false, bound = false;
  int device = -1;
};

inline int cu_rc(CUresult r) { return r == CUDA_SUCCESS ? 0 : 1000 + (int)r; }

// Driver entry points resolved at run time through the runtime API, so the
// library has no link-time dependency on libcuda (it loads on hosts without a
// driver, e.g. for the ABI checks of the CPU test suite).
struct Drv {
  bool ok = false;
  decltype(&cuDeviceGet) DeviceGet = nullptr;
  decltype(&cuDeviceGetAttribute) DeviceGetAttribute = nullptr;
  decltype(&cuMulticastGetGranularity) MulticastGetGranularity = nullptr;
  decltype(&cuMulticastCreate) MulticastCreate = nullptr;
  decltype(&cuMulticastAddDevice) MulticastAddDevice = nullptr;
  decltype(&cuMulticastBindMem) MulticastBindMem = nullptr;
  decltype(&cuMulticastUnbind) MulticastUnbind = nullptr;
  decltype(&cuMemExportToShareableHandle) MemExportToShareableHandle = nullptr;
  decltype(&cuMemImportFromShareableHandle) MemImportFromShareableHandle = nullptr;
  decltype(&cuMemGetAllocationGranularity) MemGetAllocationGranularity = nullptr;
  decltype(&cuMemCreate) MemCreate = nullptr;
  decltype(&cuMemRelease) MemRelease = nullptr;
  decltype(&cuMemAddressReserve) MemAddressReserve = nullptr;
  decltype(&cuMemAddressFree) MemAddressFree = nullptr;
  decltype(&cuMemMap) MemMap = nullptr;
  decltype(&cuMemUnmap) MemUnmap = nullptr;
  decltype(&cuMemSetAccess) MemSetAccess = nullptr;
};

template <typename F>
bool resolve(F& fn, const char* name) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPointByVersion(name, &p, 12000, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || p == nullptr) {
    cudaGetLastError();
    return false;
  }
  fn = reinterpret_cast<F>(p);
  return true;
}

const Drv& drv() {
  static Drv d;
  static bool done = false;
  if (!done) {
    done = true;
    if (cudaFree(0) != cudaSuccess) {  // runtime (and driver) initialised
      cudaGetLastError();
      return d;
    }
    bool ok = true;
#define LOMO_R(f) ok = resolve(d.f, "cu" #f) && ok
    LOMO_R(DeviceGet);
    LOMO_R(DeviceGetAttribute);
    LOMO_R(MulticastGetGranularity);
    LOMO_R(MulticastCreate);
    LOMO_R(MulticastAddDevice);
    LOMO_R(MulticastBindMem);
    LOMO_R(MulticastUnbind);
    LOMO_R(MemExportToShareableHandle);
    LOMO_R(MemImportFromShareableHandle);
    LOMO_R(MemGetAllocationGranularity);
    LOMO_R(MemCreate);
    LOMO_R(MemRelease);
    LOMO_R(MemAddressReserve);
    LOMO_R(MemAddressFree);
    LOMO_R(MemMap);
    LOMO_R(MemUnmap);
    LOMO_R(MemSetAccess);
#undef LOMO_R
    d.ok = ok;
  }
  return d;
}

#ifndef SYS_pidfd_open
#define SYS_pidfd_open 434
#endif
#ifndef SYS_pidfd_getfd
#define SYS_pidfd_getfd 438
#endif

}  // namespace lomo_peer
using namespace lomo_peer;

extern "C" {

size_t lomo_ipc_handle_bytes(void) { return sizeof(cudaIpcMemHandle_t); }

int lomo_ipc_alloc(size_t bytes, void** dev_ptr, void* handle_out) {
  if (bytes == 0 || dev_ptr == nullptr || handle_out == nullptr) return LOMO_E_ARG;
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) return (int)e;
  e = cudaMemset(p, 0, bytes);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  cudaIpcMemHandle_t h;
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    cudaFree(p);
    return (int)e;
  }
  memcpy(handle_out, &h, sizeof(h));
  *dev_ptr = p;
  return 0;
}

int lomo_ipc_open(const void* handle, void** dev_ptr) {
  if (handle == nullptr || dev_ptr == nullptr) return LOMO_E_ARG;
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  return (int)cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess);
}

int lomo_ipc_close(void* dev_ptr) {
  if (dev_ptr == nullptr) return LOMO_E_ARG;
  return (int)cudaIpcCloseMemHandle(dev_ptr);
}

int lomo_ipc_free(void* dev_ptr) {
  if (dev_ptr == nullptr) return LOMO_E_ARG;
  return (int)cudaFree(dev_ptr);
}

int lomo_peer_barrier(void* const* sig_dev, int world, int rank, int channel, uint64_t epoch,
                      int64_t timeout_ns, int* err_dev, void* stream) {
  if (sig_dev == nullptr || err_dev == nullptr || world < 1 || world > LOMO_PEER_MAX ||
      rank < 0 || rank >= world || channel < 0 || channel >= LOMO_PEER_CHANNELS || epoch == 0)
    return LOMO_E_ARG;
  k_peer_barrier<<<1, 32, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<uint64_t* const*>(const_cast<void**>(sig_dev)), world, rank, channel, epoch,
      timeout_ns, err_dev, nullptr);
  return (int)cudaGetLastError();
}

int lomo_peer_barrier_dev(void* const* sig_dev, uint64_t* epochs_dev, int world, int rank,
                          int channel, int64_t timeout_ns, int* err_dev, void* stream) {
  if (sig_dev == nullptr || epochs_dev == nullptr || err_dev == nullptr || world < 1 ||
      world > LOMO_PEER_MAX || rank < 0 || rank >= world || channel < 0 ||
      channel >= LOMO_PEER_CHANNELS)
    return LOMO_E_ARG;
  k_peer_barrier<<<1, 32, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<uint64_t* const*>(const_cast<void**>(sig_dev)), world, rank, channel, 0,
      timeout_ns, err_dev, epochs_dev);
  return (int)cudaGetLastError();
}

int lomo_mc_supported(int device) {
  const Drv& D = drv();
  if (!D.ok) return 0;
  CUdevice d;
  if (D.DeviceGet(&d, device) != CUDA_SUCCESS) return 0;
  int v = 0;
  if (D.DeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, d) != CUDA_SUCCESS)
    return 0;
  return v ? 1 : 0;
}

int lomo_mc_create(int world, size_t bytes, uint64_t* obj, size_t* granted_bytes, int* fd) {
  if (world < 1 || world > LOMO_PEER_MAX || bytes == 0 || obj == nullptr) return LOMO_E_ARG;
  const Drv& D = drv();
  if (!D.ok) return LOMO_E_UNSUPPORTED;
  CUmulticastObjectProp prop;
  memset(&prop, 0, sizeof(prop));
  prop.numDevices = (unsigned)world;
  prop.handleTypes = world > 1 ? CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR : CU_MEM_HANDLE_TYPE_NONE;
  size_t gran = 0;
  prop.size = bytes;
  CUresult r = D.MulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED);
  if (r != CUDA_SUCCESS) return r == CUDA_ERROR_NOT_SUPPORTED ? LOMO_E_UNSUPPORTED : cu_rc(r);
  prop.size = (bytes + gran - 1) / gran * gran;
  McObj* o = new (std::nothrow) McObj();
  if (o == nullptr) return LOMO_E_ARG;
  r = D.MulticastCreate(&o->mc, &prop);
  if (r != CUDA_SUCCESS) {
    delete o;
    return r == CUDA_ERROR_NOT_SUPPORTED ? LOMO_E_UNSUPPORTED : cu_rc(r);
  }
  o->have_mc = true;
  o->size = prop.size;
  if (world > 1) {
    int f = -1;
    r = D.MemExportToShareableHandle(&f, o->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
    if (r != CUDA_SUCCESS) {
      D.MemRelease(o->mc);
      delete o;
      return cu_rc(r);
    }
    o->fd = f;
  }
  if (granted_bytes) *granted_bytes = o->size;
  if (fd) *fd = o->fd;
  *obj = (uint64_t)(uintptr_t)o;
  return 0;
}

int lomo_mc_import(int pid, int fd, size_t bytes, uint64_t* obj) {
  if (pid <= 0 || fd < 0 || bytes == 0 || obj == nullptr) return LOMO_E_ARG;
  const Drv& D = drv();
  if (!D.ok) return LOMO_E_UNSUPPORTED;
  const int pidfd = (int)syscall(SYS_pidfd_open, pid, 0);
  if (pidfd < 0) return LOMO_E_UNSUPPORTED;
  const int local = (int)syscall(SYS_pidfd_getfd, pidfd, fd, 0);
  close(pidfd);
  if (local < 0) return LOMO_E_UNSUPPORTED;
  McObj* o = new (std::nothrow) McObj();
  if (o == nullptr) {
    close(local);
    return LOMO_E_ARG;
  }
  CUresult r = D.MemImportFromShareableHandle(&o->mc, (void*)(uintptr_t)local,
                                              CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
  close(local);
  if (r != CUDA_SUCCESS) {
    delete o;
    return cu_rc(r);
  }
  o->have_mc = true;
  o->size = bytes;
  *obj = (uint64_t)(uintptr_t)o;
  return 0;
}

int lomo_mc_add_device(uint64_t obj, int device) {
  McObj* o = reinterpret_cast<McObj*>((uintptr_t)obj);
  if (o == nullptr || !o->have_mc) return LOMO_E_ARG;
  const Drv& D = drv();
  CUdevice d;
  CUresult r = D.DeviceGet(&d, device);
  if (r == CUDA_SUCCESS) r = D.MulticastAddDevice(o->mc, d);
  if (r == CUDA_SUCCESS) o->device = device;
  return cu_rc(r);
}

int lomo_mc_bind(uint64_t obj, int device, void** uc_ptr, void** mc_ptr) {
  McObj* o = reinterpret_cast<McObj*>((uintptr_t)obj);
  if (o == nullptr || !o->have_mc || uc_ptr == nullptr || mc_ptr == nullptr) return LOMO_E_ARG;
  const Drv& D = drv();
  CUmemAllocationProp ap;
  memset(&ap, 0, sizeof(ap));
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = device;
  size_t gran = 0;
  CUresult r = D.MemGetAllocationGranularity(&gran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
  if (r != CUDA_SUCCESS) return cu_rc(r);
  if (o->size % gran) return LOMO_E_ARG;
  r = D.MemCreate(&o->mem, o->size, &ap, 0);
  if (r != CUDA_SUCCESS) return cu_rc(r);
  o->have_mem = true;
  r = D.MulticastBindMem(o->mc, 0, o->mem, 0, o->size, 0);
  if (r != CUDA_SUCCESS) return cu_rc(r);
  o->bound = true;
  CUmemAccessDesc acc;
  memset(&acc, 0, sizeof(acc));
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  r = D.MemAddressReserve(&o->uc_ptr, o->size, gran, 0, 0);
  if (r == CUDA_SUCCESS) r = D.MemMap(o->uc_ptr, o->size, 0, o->mem, 0);
  if (r == CUDA_SUCCESS) r = D.MemSetAccess(o->uc_ptr, o->size, &acc, 1);
  if (r != CUDA_SUCCESS) return cu_rc(r);
  r = D.MemAddressReserve(&o->mc_ptr, o->size, gran, 0, 0);
  if (r == CUDA_SUCCESS) r = D.MemMap(o->mc_ptr, o->size, 0, o->mc, 0);
  if (r == CUDA_SUCCESS) r = D.MemSetAccess(o->mc_ptr, o->size, &acc, 1);
  if (r != CUDA_SUCCESS) return cu_rc(r);
  cudaError_t e = cudaMemset((void*)o->uc_ptr, 0, o->size);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return (int)e;
  *uc_ptr = (void*)o->uc_ptr;
  *mc_ptr = (void*)o->mc_ptr;
  return 0;
}

int lomo_mc_free(uint64_t obj) {
  McObj* o = reinterpret_cast<McObj*>((uintptr_t)obj);
  if (o == nullptr) return LOMO_E_ARG;
  const Drv& D = drv();
  cudaDeviceSynchronize();
  if (o->mc_ptr) {
    D.MemUnmap(o->mc_ptr, o->size);
    D.MemAddressFree(o->mc_ptr, o->size);
  }
  if (o->uc_ptr) {
    D.MemUnmap(o->uc_ptr, o->size);
    D.MemAddressFree(o->uc_ptr, o->size);
  }
  if (o->bound) {
    CUdevice d;
    if (D.DeviceGet(&d, o->device) == CUDA_SUCCESS) D.MulticastUnbind(o->mc, d, 0, o->size);
  }
  if (o->have_mem) D.MemRelease(o->mem);
  if (o->have_mc) D.MemRelease(o->mc);
  if (o->fd >= 0) close(o->fd);
  delete o;
  return 0;
}

int lomo_mc_barrier(void* sig_mc, const void* sig_uc, int world, int channel, uint64_t epoch,
                    int64_t timeout_ns, int* err_dev, void* stream) {
  if (sig_mc == nullptr || sig_uc == nullptr || err_dev == nullptr || world < 1 ||
      world > LOMO_PEER_MAX || channel < 0 || channel >= LOMO_PEER_CHANNELS || epoch == 0)
    return LOMO_E_ARG;
  k_mc_barrier<<<1, 32, 0, (cudaStream_t)stream>>>(static_cast<uint64_t*>(sig_mc),
                                                     static_cast<const uint64_t*>(sig_uc), world,
                                                     channel, epoch, timeout_ns, err_dev, nullptr);
  return (int)cudaGetLastError();
}

int lomo_mc_barrier_dev(void* sig_mc, const void* sig_uc, uint64_t* epochs_dev, int world,
                        int channel, int64_t timeout_ns, int* err_dev, void* stream) {
  if (sig_mc == nullptr || sig_uc == nullptr || epochs_dev == nullptr || err_dev == nullptr ||
      world < 1 || world > LOMO_PEER_MAX || channel < 0 || channel >= LOMO_PEER_CHANNELS)
    return LOMO_E_ARG;
  k_mc_barrier<<<1, 32, 0, (cudaStream_t)stream>>>(static_cast<uint64_t*>(sig_mc),
                                                     static_cast<const uint64_t*>(sig_uc), world,
                                                     channel, 0, timeout_ns, err_dev, epochs_dev);
  return (int)cudaGetLastError();
}

}  // extern "C"

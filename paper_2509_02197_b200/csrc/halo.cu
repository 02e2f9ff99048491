// K15 of the C ABI: the halo exchange of a slab-decomposed stencil timestep
// over the caller's NCCL communicator (include/gfb.h, gfb_halo_exchange).
//
// The engine's own multi-GPU path (decomp.py) posts the same grouped
// send / receive through torch.distributed; this entry is for hosts that
// hold an ncclComm_t themselves. NCCL is looked up at run time: the
// libnccl.so.2 already loaded in the process (torch's, so a communicator it
// created is understood) or else the system library.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>

#include "gfb_internal.h"

namespace gfb {
namespace {

struct Nccl {
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGetErrorString) error = nullptr;
  bool ok = false;
};

const Nccl &nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    n.group_start = reinterpret_cast<decltype(&ncclGroupStart)>(dlsym(h, "ncclGroupStart"));
    n.group_end = reinterpret_cast<decltype(&ncclGroupEnd)>(dlsym(h, "ncclGroupEnd"));
    n.send = reinterpret_cast<decltype(&ncclSend)>(dlsym(h, "ncclSend"));
    n.recv = reinterpret_cast<decltype(&ncclRecv)>(dlsym(h, "ncclRecv"));
    n.error = reinterpret_cast<decltype(&ncclGetErrorString)>(dlsym(h, "ncclGetErrorString"));
    n.ok = n.group_start && n.group_end && n.send && n.recv && n.error;
  });
  return n;
}

}  // namespace
}  // namespace gfb

using namespace gfb;

extern "C" int gfb_halo_exchange(const gfb_halo_desc *d, void *nccl_comm, void *stream) {
  if (!d || d->n < 0 || d->n > GFB_MAX_HALO || !nccl_comm)
    return set_error(GFB_EINVAL, "gfb_halo_exchange: bad descriptor");
  for (int i = 0; i < d->n; ++i) {
    const gfb_halo_array &a = d->a[i];
    const bool ok = a.base && a.plane_bytes > 0 && a.width >= 0 && a.own_lo >= 0 && a.own_hi <= a.planes &&
                    a.own_hi - a.own_lo >= a.width && (d->lower < 0 || a.own_lo >= a.width) &&
                    (d->upper < 0 || a.own_hi + a.width <= a.planes);
    if (!ok) return set_error(GFB_EINVAL, "gfb_halo_exchange: bad array");
  }
  const Nccl &n = nccl();
  if (!n.ok) return set_error(GFB_EUNSUPPORTED, "gfb_halo_exchange: libnccl.so.2 not available");
  ncclComm_t comm = static_cast<ncclComm_t>(nccl_comm);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  auto plane = [](const gfb_halo_array &a, int64_t p) { return static_cast<char *>(a.base) + p * a.plane_bytes; };
  ncclResult_t r = n.group_start();
  // per neighbour: every array's send, then its receive (a peer posting the
  // same list matches them in order)
  for (int side = 0; side < 2 && r == ncclSuccess; ++side) {
    const int peer = side == 0 ? d->lower : d->upper;
    if (peer < 0) continue;
    for (int i = 0; i < d->n && r == ncclSuccess; ++i) {
      const gfb_halo_array &a = d->a[i];
      if (a.width == 0) continue;
      const size_t bytes = (size_t)(a.width * a.plane_bytes);
      const int64_t snd = side == 0 ? a.own_lo : a.own_hi - a.width;
      const int64_t rcv = side == 0 ? a.own_lo - a.width : a.own_hi;
      r = n.send(plane(a, snd), bytes, ncclChar, peer, comm, st);
      if (r == ncclSuccess) r = n.recv(plane(a, rcv), bytes, ncclChar, peer, comm, st);
    }
  }
  const ncclResult_t e = n.group_end();
  if (r == ncclSuccess) r = e;
  if (r != ncclSuccess) return set_error(GFB_ECUDA, n.error(r));
  return GFB_OK;
}

// Probe: NCCL 2.28 symmetric window at N = 1 (ncclMemAlloc + ncclCommWindowRegister + device
// ncclGetPeerPointer).  tools/nccl_probe/build.sh && ./probe
#include <cstdio>
#include <nccl.h>
#include <nccl_device.h>
__global__ void k(ncclWindow_t w, void** out) { out[0] = ncclGetPeerPointer(w, 64, 0); out[1] = ncclGetLsaPointer(w, 0, 0); }
int main() {
  ncclUniqueId id; ncclGetUniqueId(&id);
  ncclComm_t c; ncclResult_t r = ncclCommInitRank(&c, 1, id, 0); printf("init %d\n", (int)r);
  void* buf = nullptr; r = ncclMemAlloc(&buf, 1 << 20); printf("memalloc %d %p\n", (int)r, buf);
  ncclWindow_t w; r = ncclCommWindowRegister(c, buf, 1 << 20, &w, NCCL_WIN_COLL_SYMMETRIC); printf("register %d %p\n", (int)r, (void*)w);
  void** d; cudaMalloc(&d, 16); k<<<1,1>>>(w, d); void* h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("peer ptr %p (buf+64 = %p), lsa ptr %p, err %s\n", h[0], (char*)buf + 64, h[1], cudaGetErrorString(cudaGetLastError()));
  r = ncclCommWindowDeregister(c, w); printf("dereg %d\n", (int)r);
  ncclMemFree(buf); ncclCommDestroy(c);
}

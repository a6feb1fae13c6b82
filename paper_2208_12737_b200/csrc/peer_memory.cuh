// peer_memory.cuh -- peer-memory outputs for the pose-sharded path.
//
// One process per GPU on one NVLink/NVSwitch node.  The rank that collects the
// results (images, per-pose loss values and pose gradients) exports its output
// buffers once; every other rank opens them, and its kernels then store their
// rows straight into the collecting rank's HBM over NVLink.  The render and
// the gather are therefore one kernel per rank: the stores of a finished tile
// travel while the rest of the batch is still being walked, and there is no
// separate all-gather of the images afterwards (the NCCL all-gather is the
// baseline this replaces; bench.py reports both).
//
// Included by drr_kernels.cu inside its extern "C" block (uses fail()).

// cuMemGetAddressRange via the runtime's driver entry point (no -lcuda): the
// IPC handle names the whole cudaMalloc allocation, so the exporter also
// sends the pointer's offset inside it (torch's caching allocator hands out
// sub-ranges of larger segments).
typedef int (*drr_cuMemGetAddressRange_t)(unsigned long long*, size_t*, unsigned long long);

static drr_cuMemGetAddressRange_t drr_address_range_fn() {
  static drr_cuMemGetAddressRange_t fn = nullptr;
  if (fn == nullptr) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<drr_cuMemGetAddressRange_t>(p);
  }
  return fn;
}

int drr_peer_export(const void* d_ptr, drr_peer_handle* out) {
  if (d_ptr == nullptr || out == nullptr)
    return fail(DRR_ERR_INVALID_ARGUMENT, "drr_peer_export: NULL argument");
  drr_cuMemGetAddressRange_t range = drr_address_range_fn();
  if (range == nullptr) return fail(DRR_ERR_CUDA, "cuMemGetAddressRange unavailable");
  unsigned long long base = 0;
  size_t size = 0;
  const int r = range(&base, &size, reinterpret_cast<unsigned long long>(d_ptr));
  if (r != 0) return fail(DRR_ERR_INVALID_ARGUMENT, "drr_peer_export: not device memory (%d)", r);
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return fail(DRR_ERR_CUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
  static_assert(sizeof(h) == sizeof(out->ipc), "IPC handle size");
  memcpy(out->ipc, &h, sizeof(h));
  out->offset = reinterpret_cast<unsigned long long>(d_ptr) - base;
  out->bytes = size - out->offset;
  return DRR_OK;
}

int drr_peer_open(const drr_peer_handle* h, void** d_ptr) {
  if (h == nullptr || d_ptr == nullptr)
    return fail(DRR_ERR_INVALID_ARGUMENT, "drr_peer_open: NULL argument");
  cudaIpcMemHandle_t ih;
  memcpy(&ih, h->ipc, sizeof(ih));
  void* base = nullptr;
  // lazy peer access: the current device's kernels may then store into it
  const cudaError_t e = cudaIpcOpenMemHandle(&base, ih, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return fail(DRR_ERR_CUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
  *d_ptr = static_cast<char*>(base) + h->offset;
  return DRR_OK;
}

int drr_peer_close(void* d_ptr, uint64_t offset) {
  if (d_ptr == nullptr) return DRR_OK;
  const cudaError_t e = cudaIpcCloseMemHandle(static_cast<char*>(d_ptr) - offset);
  if (e != cudaSuccess) return fail(DRR_ERR_CUDA, "cudaIpcCloseMemHandle: %s", cudaGetErrorString(e));
  return DRR_OK;
}

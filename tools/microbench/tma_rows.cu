// How does the TMA tile-load time of one SM depend on the box SHAPE at equal bytes?
// One CTA per SM, one thread issues `depth` loads in flight of box {w floats, h rows} from a
// [rows][pitch] float tensor (row pitch 4352 B like the padded config-2 iterate) and waits on an
// mbarrier each; cycles per load = clock64 over `n` loads / n.   nvcc -arch=sm_100a -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(const __grid_constant__ CUtensorMap tm, int w, int h, int n, int depth, int rows_total,
                  long long* out) {
  extern __shared__ __align__(128) float smem[];
  __shared__ uint64_t bar[4];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 4; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const uint32_t bytes = uint32_t(w) * h * 4u;
  const int tile_floats = (w * h + 31) & ~31;
  uint32_t phase[4] = {0, 0, 0, 0};
  auto issue = [&](int i) {
    const int s = i % depth;
    const int y = ((blockIdx.x * 7 + i * 13) * h) % (rows_total - h);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
            "r"(smem_u32(smem + s * tile_floats)), "l"(&tm), "r"(20 + (blockIdx.x % 16) * 64), "r"(y), "r"(smem_u32(&bar[s]))
        : "memory");
  };
  for (int i = 0; i < depth; ++i) issue(i);
  const long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    const int s = i % depth;
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(smem_u32(&bar[s])),
        "r"(phase[s])
        : "memory");
    phase[s] ^= 1;
    if (i + depth < n + depth) issue(i + depth);
  }
  out[blockIdx.x] = clock64() - t0;
}

int main() {
  const int pitch = 1088, rows_total = 3 * 1042;  // padded config-2 iterate: 3 planes
  float* d;
  cudaMalloc(&d, size_t(pitch) * rows_total * 4);
  cudaMemset(d, 0, size_t(pitch) * rows_total * 4);
  long long* out;
  cudaMalloc(&out, 148 * 8);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto encode = reinterpret_cast<CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill)>(fn);
  const int shapes[][2] = {{92, 132}, {184, 66}, {64, 114}, {128, 57}, {256, 28}, {92, 66}, {92, 33}, {32, 132}};
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (auto& sh : shapes) {
    const int w = sh[0], h = sh[1];
    CUtensorMap tm;
    const cuuint64_t dims[2] = {cuuint64_t(pitch), cuuint64_t(rows_total)};
    const cuuint64_t strides[1] = {cuuint64_t(pitch) * 4};
    const cuuint32_t box[2] = {cuuint32_t(w), cuuint32_t(h)};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", int(r)); continue; }
    for (int depth : {1, 2}) {
      const int n = 400;
      const size_t smem = size_t(((w * h + 31) & ~31)) * 4 * depth + 128;
      k<<<148, 32, smem>>>(tm, w, h, n, depth, rows_total, out);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("launch failed: %s\n", cudaGetErrorString(e)); return 1; }
      std::vector<long long> hst(148);
      cudaMemcpy(hst.data(), out, 148 * 8, cudaMemcpyDeviceToHost);
      std::sort(hst.begin(), hst.end());
      const double cyc = double(hst[74]) / n;
      printf("box %3d x %3d (%5.1f KB) depth %d: %7.0f cycles per load, %5.1f B/clk/SM, %5.1f cycles per row\n", w, h,
             w * h * 4 / 1024.0, depth, cyc, w * h * 4 / cyc, cyc / h);
    }
  }
  return 0;
}

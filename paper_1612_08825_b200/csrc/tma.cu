// Host-side tensor-map encoding (cuTensorMapEncodeTiled via cudart's driver
// entry point lookup).
#include <cudaTypedefs.h>

#include "common.cuh"
#include "tma.cuh"

namespace ct {

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    else
      cudaGetLastError();
  }
  return fn;
}

bool encode_tmap_2d(CUtensorMap* map, const void* base, int esz, uint64_t cols, uint64_t rows,
                    uint32_t box_cols, uint32_t box_rows) {
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0) return false;
  if ((cols * esz) % 16 != 0) return false;
  if ((box_cols * esz) % 16 != 0 || box_cols > 256 || box_rows > 256) return false;
  // TMA tensor coordinates are signed 32-bit: callers pass row indices as int,
  // so a taller view must fall back to the plain-load kernels
  if (rows >= (1ull << 31) || cols >= (1ull << 31)) return false;
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * (cuuint64_t)esz};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, esz == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                  const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool encode_tmap_3d(CUtensorMap* map, const void* base, int esz, uint64_t d0, uint64_t d1, uint64_t d2,
                    uint32_t box0, uint32_t box1) {
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0) return false;
  if ((d0 * esz) % 16 != 0 || (box0 * esz) % 16 != 0 || box0 > 256 || box1 > 256) return false;
  if (d0 >= (1ull << 31) || d1 >= (1ull << 31) || d2 >= (1ull << 31)) return false;  // s32 coordinates
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {d0 * (cuuint64_t)esz, d0 * d1 * (cuuint64_t)esz};
  cuuint32_t box[3] = {box0, box1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, esz == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                  const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool encode_tmap_4d(CUtensorMap* map, const void* base, int esz, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t d3,
                    uint32_t box0, uint32_t box1) {
  if ((reinterpret_cast<uintptr_t>(base) & 15) != 0) return false;
  if ((d0 * esz) % 16 != 0 || (box0 * esz) % 16 != 0 || box0 > 256 || box1 > 256) return false;
  if (d0 >= (1ull << 31) || d1 >= (1ull << 31) || d2 >= (1ull << 31) || d3 >= (1ull << 31)) return false;
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {d0, d1, d2, d3};
  cuuint64_t strides[3] = {d0 * (cuuint64_t)esz, d0 * d1 * (cuuint64_t)esz, d0 * d1 * d2 * (cuuint64_t)esz};
  cuuint32_t box[4] = {box0, box1, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(map, esz == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4,
                  const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

}  // namespace ct

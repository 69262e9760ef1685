// render.h — the limit case of the compositing and the VDI renderers (render.cu).
// Product code (sm_100a).  Shares nothing with oracle/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"

namespace vdi {

struct CamF {
  float eye[3], fwd[3], right[3], up[3];
  float tan_x, tan_y;
};

// novel-view rendering of a full-representation VDI of W x H lists (k slots)
struct NovelParams {
  const uint8_t* count;  // [H*W]
  const float2* depth;   // [H*W][k]
  const float4* rgba;    // [H*W][k]
  uint32_t W, H;
  int k;
  CamF gen, view;        // generation camera of the VDI, camera of the new view
  float half[3];         // the volume's world box [-half, half]
  float dt;              // march step (one voxel, world units)
  uint32_t W_out, H_out;
  float4* out;           // [H_out*W_out] premultiplied RGBA
};

cudaError_t launch_image(const MergeParams& mp, float4* out, cudaStream_t st);
cudaError_t launch_gen_view(const uint8_t* count, const float4* rgba, uint32_t P, int k, float4* out, cudaStream_t st);
cudaError_t launch_novel_view(const NovelParams& np, cudaStream_t st);
cudaError_t launch_rows_push(const float4* src, float4* dst, uint32_t n, uint32_t blocks, uint32_t* flag,
                             cudaStream_t st);
cudaError_t preload_render();

}  // namespace vdi

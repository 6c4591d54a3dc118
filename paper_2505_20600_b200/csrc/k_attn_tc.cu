// k_attn_tc.cu — tcgen05 varlen FMHA (placeholder until the tensor-core kernel lands).
#include "kernels.h"
namespace ig {
void launch_attn_tc(const AttnArgs& a, cudaStream_t st) { launch_attn_simt<bf16>(a, st); }
}  // namespace ig

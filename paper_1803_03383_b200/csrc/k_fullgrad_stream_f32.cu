// K1 streaming kernel, f32 instantiations (see the end of k_fullgrad_stream.cu)
#define HALP_STREAM_TU 1
#include "k_fullgrad_stream.cu"

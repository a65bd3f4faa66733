// gc_predict_ref.cu -- the reference-arithmetic instantiations of gc_predict.cu
// (k_predict<MODE_REF, K>, k_propagate_step, gc_propagate_step), compiled with
// --fmad=false so ptxas never contracts a multiply into a following add: the packed
// FP32x2 operations of exp_np2 / ref_logit2 must round exactly like numpy's float32 ops.
#define GC_PREDICT_REF_TU 1
#include "gc_predict.cu"

/*
 * canvas_post.h — C ABI of the post-pass of a replaced conv
 * (libcanvas_post.so): training-mode BatchNorm2d over the Canvas kernel's
 * output with the block's ReLU and residual add fused in, and the stem
 * max-pool of the ResNet backbones (deterministic gather backward).
 *
 * What it replaces in the reference:
 *   SPEC.md:658 (trainer_plugin.build_module, "BN post-pass" after the FC of
 *   a built module) and, in the network path, the
 *   backbone BatchNorm2d that follows every replaced nn.Conv2d; the reference
 *   specifies both but ships no numeric code.
 *   Semantics are torch.nn.functional.batch_norm(training=True) followed by
 *   (+ residual) and ReLU: biased variance for normalisation, unbiased for the
 *   running variance, running = (1 - momentum) * running + momentum * batch.
 *
 * Conventions: fp32, contiguous [N, C, H*W] device tensors owned by the
 * caller; `workspace` holds canvas_bn_workspace() bytes of per-slice
 * partials; calls only enqueue kernels on `stream` (no allocation, no sync;
 * CUDA-graph capturable).  Deterministic: no atomics.  0 = OK, negative =
 * error (message from canvas_post_last_error, thread-local).
 */
#ifndef CANVAS_POST_H
#define CANVAS_POST_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CANVAS_POST_ABI_VERSION 2
#define CANVAS_POST_OK 0
#define CANVAS_POST_ERR_ARGS (-5)
#define CANVAS_POST_ERR_CUDA (-4)

int canvas_post_abi_version(void);

/* Bytes of workspace a BN forward or backward call at this shape needs. */
size_t canvas_bn_workspace(int64_t N, int64_t C, int64_t HW);

/* y = act(bn(x) [+ residual]); act = ReLU when relu != 0.  running_mean /
 * running_var may both be NULL (no running-stat update).  Writes the batch
 * mean and 1/sqrt(var + eps) to save_mean / save_invstd for the backward, and,
 * when relu_mask is non-NULL (relu != 0), one byte (y > 0) per element. */
int canvas_bn_forward(int64_t N, int64_t C, int64_t HW, const float* x, const float* residual, float* y,
                      const float* gamma, const float* beta, float* running_mean, float* running_var,
                      float* save_mean, float* save_invstd, float momentum, float eps, int relu, uint8_t* relu_mask,
                      void* workspace, void* stream);

/* dx (and dresidual = the gradient reaching the residual, when non-NULL),
 * dgamma, dbeta (written, not accumulated) from dy = dL/dy.  The ReLU mask
 * (relu'(0) = 0) comes from relu_mask (the forward's bytes) when non-NULL,
 * else from y > 0 (the forward output); both may be NULL when relu == 0. */
int canvas_bn_backward(int64_t N, int64_t C, int64_t HW, const float* x, const float* y, const uint8_t* relu_mask,
                       const float* dy, const float* gamma, const float* save_mean, const float* save_invstd,
                       float* dx, float* dresidual, float* dgamma, float* dbeta, int relu, void* workspace,
                       void* stream);

/* Max-pool (square window K, stride S, padding P, no dilation, floor mode) of
 * [N, C, H, W]: y [N, C, OH, OW] and the winner's window slot (kh*K + kw, one
 * byte per output; first maximum in row-major order, NaN propagates). */
int canvas_maxpool2d_forward(int64_t N, int64_t C, int64_t H, int64_t W, int K, int S, int P, const float* x, float* y,
                             uint8_t* argmax, void* stream);

/* dx [N, C, H, W] (written) from dy [N, C, OH, OW] and the forward's argmax. */
int canvas_maxpool2d_backward(int64_t N, int64_t C, int64_t H, int64_t W, int K, int S, int P, const float* dy,
                              const uint8_t* argmax, float* dx, void* stream);

const char* canvas_post_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* CANVAS_POST_H */

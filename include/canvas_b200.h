/*
 * canvas_b200.h — C ABI of the B200 executor for Canvas kernel graphs
 * (arXiv 2304.07741).  libcanvas_b200.so exports exactly these symbols.
 *
 * What each entry point replaces in the reference (/root/reference):
 *
 *   The reference ships NO numeric executor for a sampled kernel: its
 *   interpreter (SPEC.md:491-533 `interpreter.execute`) and trainer plugin
 *   (SPEC.md:628-667 `trainer_plugin.build_module`, forward/backward of the
 *   kernel-graph-to-module replacement) are specified but not
 *   shipped.  The boundary payload they consume IS shipped:
 *   `canvas-ir v1` text (pkg/src/canvas/ir.py:3-16, `emit` :68-89, `parse`
 *   :97-169) plus a target assignment (`TargetSolution.assignment`,
 *   ir.py:48-53).  The Python side (paper_2304_07741_b200.lowering) parses
 *   that payload with the reference-compatible front end and flattens it to
 *   a POD "plan blob"; these functions execute it.
 *
 *   canvas_plan_create   <- build_module(ir, assignment)
 *   canvas_plan_query    <- (allocation sizing; new)
 *   canvas_forward       <- module.forward == interpreter.execute
 *                                                              SPEC.md:502-510, 646-650
 *   canvas_backward      <- autograd of the module
 *   canvas_last_error    <- the reference raises ValueError subclasses
 *                           (IrError ir.py:31, NotApplicable primitives.py:51,
 *                           ShapeMismatch micro_dag.py:37, NonIntegral
 *                           shape_algebra.py:43-56); here a negative code +
 *                           message, raised as exceptions again in Python.
 *
 * Conventions: all tensors are fp32, contiguous, caller-owned device memory
 * laid out as SURVEY App. A.0 ([N, C, H, W] at the module boundary).  After
 * canvas_plan_create the library performs no device allocation, no host
 * synchronisation and no host callback: every call only enqueues kernels on
 * `stream`, so calls are CUDA-graph capturable.  fc_dw is written, not
 * accumulated.  Identical inputs give bitwise-identical outputs (no atomics).
 * Plans are immutable; concurrent calls on different streams with distinct
 * workspace/saved buffers are safe.
 */
#ifndef CANVAS_B200_H
#define CANVAS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CANVAS_OK 0
#define CANVAS_ERR_BLOB (-1)     /* malformed plan blob */
#define CANVAS_ERR_VERSION (-2)  /* blob ABI version mismatch */
#define CANVAS_ERR_COMPILE (-3)  /* NVRTC compilation of the plan failed */
#define CANVAS_ERR_CUDA (-4)     /* CUDA driver error (launch, module load) */
#define CANVAS_ERR_ARGS (-5)     /* null/size mismatch in call arguments */
#define CANVAS_ERR_DEVICE (-6)   /* device is not sm_100 (no fallback exists) */

typedef struct canvas_plan canvas_plan; /* opaque; immutable after create */

/* ABI version of the blob format this library accepts. */
int canvas_abi_version(void);

/* Parse + compile a plan blob (lowering.Plan.blob()) for `cuda_device`. */
int canvas_plan_create(const void* blob, size_t nbytes, int cuda_device, canvas_plan** out);

void canvas_plan_destroy(canvas_plan* p);

/* Buffer sizes at batch `batch`: forward scratch (always 0 in v1),
 * `saved` (forward activations kept for backward, all replicas), and
 * backward workspace.  Every tensor inside `saved` / the workspace sits between
 * two 16 KB guard zones (included in these sizes), so vectorised kernels may
 * read whole 16-byte chunks across a tensor edge; callers just pass the start
 * of the buffers they allocated. */
int canvas_plan_query(const canvas_plan* p, int64_t batch, size_t* fwd_workspace, size_t* saved_bytes,
                      size_t* bwd_workspace);

/* Kernel launches one canvas_forward (phase 0) / canvas_backward (phase 1)
 * enqueues, counting every replica. */
int canvas_plan_launches(const canvas_plan* p, int phase);

/* y = kernel(x) for every Fig.-2 replica.  fc_w holds n_fc device pointers
 * (replica-major, IR edge order, each [out, prod(in ch)] row-major).
 * Launch records of blob kind 2 issue 16-byte vector accesses: every tensor
 * pointer they receive must be 16-byte aligned (CANVAS_ERR_ARGS otherwise;
 * PyTorch allocations always are). */
int canvas_forward(const canvas_plan* p, int64_t batch, const float* x, const float* const* fc_w, int n_fc,
                   float* y, void* saved, void* workspace, void* stream);

/* dx, fc_dw from dy and the `saved` buffer written by the matching forward. */
int canvas_backward(const canvas_plan* p, int64_t batch, const float* x, const float* const* fc_w, int n_fc,
                    const void* saved, const float* dy, float* dx, float* const* fc_dw, void* workspace,
                    void* stream);

/* Measurement hook: record CUDA events (CUevent / cudaEvent_t handles,
 * 2*n_pairs of them, start/end interleaved) around every launch of launch
 * record `record`, cycling through the pairs; several records may be
 * profiled at once; n_pairs = 0 disables that record.  Used by bench.py to
 * time kernels inside a full training step. */
int canvas_plan_profile(canvas_plan* p, int record, void* const* events, int n_pairs);

/* Launches of `record` recorded since its canvas_plan_profile. */
int64_t canvas_plan_profile_count(const canvas_plan* p, int record);

/* Message of the last failing call on this thread. */
const char* canvas_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* CANVAS_B200_H */

// ds_graph.cu -- the CG solve as ONE graph launch: a CUDA graph with a WHILE
// conditional node whose body holds K captured CG iterations followed by a
// 1-thread kernel that sets the loop condition to (s->done == 0).  The host
// enqueues the setup, launches the graph and reads the result once: no
// scalar readbacks between iterations and no post-convergence no-op steps
// beyond the body's K - 1 (solver.py:102-116 loop, run on the device).
#include "ds_common.cuh"

namespace ds {

__global__ void cg_while_continue_kernel(cudaGraphConditionalHandle h, const ds_cg_scalars* s) {
  cudaGraphSetConditional(h, s->done == 0 ? 1u : 0u);
}

}  // namespace ds

using namespace ds;

extern "C" int ds_while_graph_begin(void* stream, void** graph_out,
                                    unsigned long long* handle_out) {
  *graph_out = nullptr;
  cudaGraph_t g = nullptr;
  DS_CUDA(cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  cudaError_t e = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
  cudaGraphNodeParams p = {};
  cudaGraphNode_t node;
  if (e == cudaSuccess) {
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    e = cudaGraphAddNode(&node, g, nullptr, 0, &p);
  }
  if (e == cudaSuccess)
    e = cudaStreamBeginCaptureToGraph(as_stream(stream), p.conditional.phGraph_out[0], nullptr,
                                      nullptr, 0, cudaStreamCaptureModeRelaxed);
  if (e != cudaSuccess) {
    cudaGraphDestroy(g);
    return cuda_fail(e, "while-graph begin");
  }
  *graph_out = g;
  *handle_out = (unsigned long long)h;
  return DS_OK;
}

extern "C" int ds_cg_while_continue(unsigned long long handle, const ds_cg_scalars* s,
                                    void* stream) {
  cg_while_continue_kernel<<<1, 1, 0, as_stream(stream)>>>((cudaGraphConditionalHandle)handle, s);
  DS_LAUNCH_CHECK("cg_while_continue_kernel");
  return DS_OK;
}

extern "C" int ds_while_graph_end(void* stream, void* graph, void** exec_out) {
  *exec_out = nullptr;
  cudaGraph_t body = nullptr;
  cudaError_t e = cudaStreamEndCapture(as_stream(stream), &body);
  cudaGraphExec_t ex = nullptr;
  if (e == cudaSuccess) e = cudaGraphInstantiate(&ex, static_cast<cudaGraph_t>(graph), 0);
  if (e != cudaSuccess) return cuda_fail(e, "while-graph end / instantiate");
  *exec_out = ex;
  return DS_OK;
}

extern "C" int ds_graph_exec_launch(void* exec, void* stream) {
  DS_CUDA(cudaGraphLaunch(static_cast<cudaGraphExec_t>(exec), as_stream(stream)));
  return DS_OK;
}

extern "C" int ds_graph_destroy(void* graph, void* exec) {
  if (exec) DS_CUDA(cudaGraphExecDestroy(static_cast<cudaGraphExec_t>(exec)));
  if (graph) DS_CUDA(cudaGraphDestroy(static_cast<cudaGraph_t>(graph)));
  return DS_OK;
}

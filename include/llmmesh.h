/* llmmesh.h — C ABI of the B200 LLM-Mesh control plane (libllmmesh.so).
 *
 * Drop-in for the reference's proj/include/llmmesh.h:17-56: same opaque
 * handle, entry points, status codes and ownership rules, so the reference
 * CLI and any FFI binding link against this library unchanged
 * (see INTEGRATION.md). Extensions for the B200 build are at the end.
 *
 *   status   0 OK / 1 ERR_ARG / 2 ERR_CONFIG / 3 ERR_RUNTIME  (capi.cpp:40-51)
 *   open     allocates the handle; close frees it; the config file is read
 *            lazily at run/compare so overrides can be applied first
 *   error    message of the last failed call, owned by the handle
 *   threads  a handle is not thread-safe; the engine is single-threaded
 */
#ifndef LLMMESH_H
#define LLMMESH_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct llm_experiment llm_experiment;

typedef enum llm_status { LLM_OK = 0, LLM_ERR_ARG = 1, LLM_ERR_CONFIG = 2, LLM_ERR_RUNTIME = 3 } llm_status;

const char* llm_version(void);
llm_status llm_experiment_open(const char* config_path, llm_experiment** out);
/* dotted-path override; the value parses as JSON, else as a string */
llm_status llm_experiment_set(llm_experiment* exp, const char* key, const char* value);
llm_status llm_experiment_set_seed(llm_experiment* exp, uint64_t seed);
llm_status llm_experiment_set_output_dir(llm_experiment* exp, const char* dir);
/* summary.json, requests.csv, ttft_cdf.csv, effective_config.json (+ events.jsonl) */
llm_status llm_experiment_run(llm_experiment* exp);
/* comma-separated policies (mesh,exclusive,exclusive_cpu): per-policy dirs + comparison.json */
llm_status llm_experiment_compare(llm_experiment* exp, const char* policies_csv);
/* plain names after run, "<policy>.<name>" after compare */
llm_status llm_experiment_metric(const llm_experiment* exp, const char* name, double* out);
const char* llm_experiment_error(const llm_experiment* exp);
void llm_experiment_close(llm_experiment* exp);

/* ---- B200 build extensions ------------------------------------------------
 * capture: run the configured policy and write the parity artifacts
 *   (events.jsonl, ops.csv ScaleOp transcript, steps.csv launched plans,
 *   hash.txt state hash, plus the run outputs) into `dir`.
 * attach_gpu: execute every priced action on B200s through libmesh_gpu.so
 *   (dlopen'ed from `gpu_lib_path`): cluster node i runs on CUDA device
 *   devices[i % n_devices]. Decisions stay those of the virtual-time
 *   schedule (parity mode); tokens are produced by the GPU. Extra metrics:
 *   "gpu.steps", "gpu.decode_tokens", "gpu.prefill_tokens", "gpu.device_ms",
 *   "gpu.swap_out_bytes", "gpu.migrate_bytes", "gpu.blocks_moved". */
llm_status llm_experiment_capture(llm_experiment* exp, const char* dir);
llm_status llm_experiment_attach_gpu(llm_experiment* exp, const char* gpu_lib_path, const int32_t* devices,
                                     int32_t n_devices, int64_t kv_pool_bytes);

#ifdef __cplusplus
}
#endif

#endif /* LLMMESH_H */

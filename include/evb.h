/*
 * evb.h — C ABI of the B200-native SEvoBench hot path (libevb.so).
 *
 * Plain C: opaque handles, plain pointers and sizes, integer status codes,
 * a thread-local last-error string, and an explicit cudaStream_t (passed as
 * void*) on every device call. No exception crosses this boundary and no
 * torch type appears in it. Status codes map onto the reference's error
 * conventions:
 *
 *   EVB_ERR_INVALID_ARGUMENT  -> std::invalid_argument  (problems/instance.hpp:222-223,
 *                                                       problems/batch.hpp:250-252)
 *   EVB_ERR_CONFIG            -> evobench::config_error (common.hpp:12-15, 25-28)
 *   EVB_ERR_LOGIC             -> std::logic_error       (de/engine.hpp:32-33)
 *   EVB_ERR_RUNTIME           -> std::runtime_error     (CUDA / allocation failures)
 *
 * All file:line citations point into the reference tree
 * (/root/reference/proj/include/evobench/...).  There is no CPU fallback:
 * every compute entry point launches sm_100a kernels or fails.
 */
#ifndef EVB_H_
#define EVB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EVB_ABI_VERSION 1

#if defined(__GNUC__)
#define EVB_API __attribute__((visibility("default")))
#else
#define EVB_API
#endif

enum evb_status {
  EVB_OK = 0,
  EVB_ERR_INVALID_ARGUMENT = 1,
  EVB_ERR_CONFIG = 2,
  EVB_ERR_LOGIC = 3,
  EVB_ERR_RUNTIME = 4
};

/* Arithmetic type of a problem / engine: the reference's template parameter T. */
enum evb_dtype { EVB_F32 = 0, EVB_F64 = 1 };

/* Same order as evobench::problems::base_kind (problems/functions.hpp:15-26). */
enum evb_base_kind {
  EVB_SPHERE = 0,
  EVB_ELLIPTIC = 1,
  EVB_BENT_CIGAR = 2,
  EVB_DISCUS = 3,
  EVB_ROSENBROCK = 4,
  EVB_RASTRIGIN = 5,
  EVB_ACKLEY = 6,
  EVB_GRIEWANK = 7,
  EVB_SCHWEFEL_12 = 8,
  EVB_EXPANDED_SCHAFFER_F6 = 9
};

typedef struct evb_problem_s* evb_problem; /* immutable device-resident problem_instance */
typedef struct evb_scratch_s* evb_scratch; /* per-task evaluation scratch (eval_scratch)   */

/* ---- library ---------------------------------------------------------------------- */

EVB_API int evb_abi_version(void);
/* Message of the last failing call on this thread ("" if none). */
EVB_API const char* evb_last_error(void);
/* Device properties the kernels size themselves by (SM count, smem/SM, L2 bytes). */
EVB_API int evb_device_info(int device, int* sm_count, int* smem_per_sm, int* l2_bytes, int* cc_major,
                    int* cc_minor);

/* Device memory helpers for hosts without a CUDA toolchain (FFI bindings, the C++ wrapper). */
EVB_API int evb_device_alloc(size_t bytes, void** out);
EVB_API int evb_device_free(void* ptr);
EVB_API int evb_copy_to_device(void* dst, const void* src_host, size_t bytes);
EVB_API int evb_copy_to_host(void* dst_host, const void* src, size_t bytes);
EVB_API int evb_synchronize(void);

/* ---- problems (problems/instance.hpp:180-252) -------------------------------------- */

/* Shifted-rotated base problem: value(x) = base(M (x - o)) + bias, rosenbrock on z + 1
 * (problems/instance.hpp:221-228, 82-91). shift (dim) and rotation (dim*dim, row-major)
 * are HOST pointers of the problem dtype; they are copied to the device once. */
EVB_API int evb_problem_create_base(int dtype, int dim, int kind, const void* shift,
                            const void* rotation, double bias, evb_problem* out);

/* Hybrid problem (problems/instance.hpp:97-112, 229-231): z = M (x - o), permute, split into
 * chunks, sum per-chunk base values, plus bias. */
EVB_API int evb_problem_create_hybrid(int dtype, int dim, const void* shift, const void* rotation,
                              double bias, int n_chunks, const int* sub_kinds,
                              const int* chunk_sizes, const int* permutation, evb_problem* out);

/* Composition problem (problems/instance.hpp:116-174, 232): n_comp components, each with its
 * own shift (n_comp*dim) and rotation (n_comp*dim*dim), sigma, lambda and bias. */
EVB_API int evb_problem_create_composition(int dtype, int dim, int n_comp, const int* kinds,
                                   const void* shifts, const void* rotations,
                                   const double* sigma, const double* lambda,
                                   const double* comp_bias, double bias, evb_problem* out);

EVB_API int evb_problem_destroy(evb_problem p);
EVB_API int evb_problem_dim(evb_problem p);
EVB_API int evb_problem_dtype(evb_problem p);

/* ---- scratch (problems/instance.hpp:45-56) ----------------------------------------- */

EVB_API int evb_scratch_create(evb_scratch* out);
EVB_API int evb_scratch_destroy(evb_scratch s);
/* Page-locked host staging owned by the scratch (grown on demand, freed with it): the C++
 * wrapper flattens a std::vector<std::vector<T>> batch into it so evb_evaluate_batch_host runs
 * at full host-link bandwidth and writes the fitness values into it directly.  Replaces the
 * per-call heap flatten of problems::evaluate_batch's AoS input (problems/batch.hpp:243-247). */
EVB_API int evb_scratch_host_staging(evb_scratch s, size_t bytes, void** out);

/* ---- batched evaluation (problems/batch.hpp:243-278) ------------------------------- */

/* out[b] = problem.evaluate(X[b]) for b < n_points.  X and out are DEVICE pointers of the
 * problem dtype; X is row-major with row stride ldx elements (ldx >= dim).  n_points == 0
 * is valid and launches nothing (problems/batch.hpp:247-249).  ldx < dim is the analogue of
 * the reference's dimension mismatch -> EVB_ERR_INVALID_ARGUMENT. */
EVB_API int evb_evaluate_batch(evb_problem p, evb_scratch s, const void* X, int64_t n_points,
                       int64_t ldx, void* out, void* stream);

/* Several base kinds on ONE z = M (x - o) (BASELINE config 1: "three transforms are
 * evaluated on the same z").  Base problems only; kinds[k] in {sphere, elliptic, bent_cigar,
 * discus, rastrigin, ackley, griewank}; out[k*ldo + b] = base_k(z_b) + biases[k]. */
EVB_API int evb_evaluate_batch_multi(evb_problem p, evb_scratch s, int n_kinds, const int* kinds,
                             const double* biases, const void* X, int64_t n_points,
                             int64_t ldx, void* out, int64_t ldo, void* stream);

/* Host-buffer form (batched_evaluate, problems/batch.hpp:281-288): X_host (n_points*ldx) and
 * out_host (n_points) are host memory; the call copies in, evaluates and copies out on the
 * scratch's own streams and returns when out_host is filled.  For the fused fp64 GEMM path the
 * copy of X is split into column chunks that the kernel consumes as they land (copy/compute
 * overlap; EVB_H2D_CHUNKS, default 4, halving widths); page-locked out_host is written by the
 * kernel directly.  Pinned X_host gives full host-link bandwidth. */
EVB_API int evb_evaluate_batch_host(evb_problem p, evb_scratch s, const void* X_host, int64_t n_points,
                            int64_t ldx, void* out_host);
/* One device population on several problems (same dimension and dtype): outs[k] (device,
 * n_points) receives problem k's fitness.  Two or three fp64 base problems with fused kinds run
 * as ONE launch whose stages carry X once for all problems; otherwise one launch per problem.
 * Replaces several problems::evaluate_batch calls on one population (problems/batch.hpp:243-278,
 * e.g. a suite's problems at one generation's population); results equal one call per problem. */
EVB_API int evb_evaluate_batch_problems(const evb_problem* problems, int n_problems, evb_scratch s, const void* X,
                                        int64_t n_points, int64_t ldx, void* const* outs, void* stream);

/* One host population on several problems (same dimension and dtype): X crosses the host link
 * once — overlapped with the first problem's fused GEMM — and every problem is evaluated on the
 * resident copy; out_host[k] (n_points values) receives problem k's fitness.  Equivalent to
 * n_problems evb_evaluate_batch_host calls, with one H2D copy instead of n_problems. */
EVB_API int evb_evaluate_batch_host_many(const evb_problem* problems, int n_problems, evb_scratch s,
                                         const void* X_host, int64_t n_points, int64_t ldx,
                                         void* const* out_host);

/* ---- random words (core/rng.hpp:37-121) --------------------------------------------- */

/* PHILOX: counter-based Philox4x32-10 words.  word(key, ctr_hi, n) = lanes (2(n&1), 2(n&1)+1)
 * of block n>>1 under counter (lo(n>>1), hi(n>>1), lo(ctr_hi), hi(ctr_hi)).  Engines give each
 * (generation g, individual i) its own sub-stream ctr_hi = (g << 32) | i (archive victims:
 * sub 0xFFFFFFFF, init_population: 0xFFFFFFF0), so every individual draws in parallel; the words
 * each individual consumed are exported (evb_de_last_draws) so the reference engine can replay
 * them in its own sequential order through rng_stream::scripted (core/rng.hpp:54-58).
 * WORDS: oracle mode — a caller-supplied word list consumed strictly in the reference's order
 * (e.g. the raw words of rng_stream(42, 0)), reproducing the reference run exactly. */
enum evb_rng_mode { EVB_RNG_PHILOX = 0, EVB_RNG_WORDS = 1 };
typedef struct evb_rng_s* evb_rng;

EVB_API int evb_rng_create_philox(uint64_t key, evb_rng* out);
EVB_API int evb_rng_create_words(const uint64_t* words_host, int64_t n_words, evb_rng* out);
EVB_API int evb_rng_destroy(evb_rng r);
/* Synchronous: WORDS cursor (next unread word), PHILOX generation counter, overflow flag. */
EVB_API int evb_rng_state(evb_rng r, int64_t* cursor, uint32_t* generation, int* overflow);
EVB_API int evb_rng_set_generation(evb_rng r, uint32_t generation);
/* n device-generated Philox words (key, ctr_hi, start..start+n) into host memory. */
EVB_API int evb_philox_words(uint64_t key, uint64_t ctr_hi, uint64_t start, int64_t n, uint64_t* out_host);

/* ---- best-so-far recorder (experiment/recorder.hpp:35-155) ------------------------------ */

/* Device-resident best_so_far_record: n_runs x (max_fes / interval) checkpoints; slot k holds the
 * running minimum after exactly (k+1)*interval evaluations; finish() fills a stopped run's tail. */
typedef struct evb_recorder_s* evb_recorder;
EVB_API int evb_recorder_create(int dtype, int n_runs, int64_t max_fes, int64_t interval, evb_recorder* out);
EVB_API int evb_recorder_destroy(evb_recorder r);
EVB_API int evb_recorder_checkpoints(evb_recorder r);
/* on_evaluate for n device values of `run`, in FE order */
EVB_API int evb_recorder_observe(evb_recorder r, int run, const void* values, int64_t n, void* stream);
/* on_run_end for runs [run0, run0 + n) */
EVB_API int evb_recorder_finish(evb_recorder r, int run0, int n, void* stream);
EVB_API int evb_recorder_grid(evb_recorder r, void* grid_host, int64_t* fes_host);
/* to_csv (recorder.hpp:103-121) for runs laid out problem x instance x run (run fastest); call
 * with buf = NULL to get the length in *len. */
EVB_API int evb_recorder_csv(evb_recorder r, const char* suite_name, int dim, int n_problems,
                             const int* problem_ids, int instances, int runs, char* buf, int64_t cap,
                             int64_t* len);

/* ---- parameter_record (experiment/parameter_record.hpp:15-95) ------------------------------- */

/* Per run, the (generation, mu_F, mu_CR) series an adaptive DE engine reports after each
 * generation (de/engine.hpp:126-129 on_generation; JADE: mu, SHADE: memory means). */
typedef struct evb_param_trace_s* evb_param_trace;

EVB_API int evb_param_trace_create(int dtype, int n_runs, int capacity, evb_param_trace* out);
EVB_API int evb_param_trace_destroy(evb_param_trace t);
/* run `run`'s series (up to cap entries; *count = entries recorded; mu arrays in the dtype) */
EVB_API int evb_param_trace_get(evb_param_trace t, int run, int* generations, void* mu_f, void* mu_cr, int cap,
                                int* count);
/* parameter_record::to_csv (problem,instance,run,generation,mu_f,mu_cr), runs laid out
 * problem-major, run index fastest; *len = full length (buf may be NULL). */
EVB_API int evb_param_trace_csv(evb_param_trace t, int n_problems, const int* problem_ids, int instances, int runs,
                                char* buf, int64_t cap, int64_t* len);

/* ---- DE engine (de/engine.hpp:51-173, de/builder.hpp:16-78) --------------------------- */

/* strategy slots, by the reference's names (de/strategy.hpp, de/parameter.hpp) */
enum evb_de_mutation { EVB_MUT_RAND1 = 0 /* "rand_1" */, EVB_MUT_BEST1 = 1 /* "best_1" */,
                       EVB_MUT_TTPB1 = 2 /* "ttpb_1" */ };
enum evb_de_crossover { EVB_CX_BINOMIAL = 0 /* "binomial" */, EVB_CX_EXPONENTIAL = 1 /* "exponential" */ };
enum evb_de_repair { EVB_REP_CLIP = 0 /* "clip" */, EVB_REP_REFLECT = 1 /* "reflect" */,
                     EVB_REP_MIDPOINT_TARGET = 2 /* "midpoint_target" */,
                     EVB_REP_REINITIALIZE = 3 /* "reinitialize" */ };
enum evb_de_parameter { EVB_PAR_FIXED = 0 /* "fixed" */, EVB_PAR_JADE = 1 /* "jade" */,
                        EVB_PAR_SHADE = 2 /* "shade" */ };

typedef struct {
  int mutation, crossover, repair, parameter;
  double f, cr;        /* fixed_parameter(F, CR)                 de/parameter.hpp:79-97   */
  double p_best;       /* ttpb1_mutation(p, use_archive)         de/strategy.hpp:124-165  */
  int use_archive;
  int memory_size;     /* shade_parameter(H)                     de/parameter.hpp:149-213 */
  double jade_c;       /* jade_parameter(c)                      de/parameter.hpp:99-147  */
  double archive_rate; /* de_builder::archive_rate               de/builder.hpp:44-48     */
  int reduction;       /* population_policy: 0 fixed, 1 linear_reduction(N_init = pop_size, n_min)
                          de/policy.hpp:14-60 (L-SHADE)                                       */
  int n_min;
} evb_de_config;

enum evb_de_policy { EVB_POP_FIXED = 0 /* "fixed" */, EVB_POP_LINEAR_REDUCTION = 1 /* "linear_reduction" */ };

typedef struct evb_de_s* evb_de;

/* Validates like de_builder::build + de_engine::validate_run; unknown slots -> EVB_ERR_CONFIG
 * (there is no CPU fallback for a strategy without a GPU kernel). */
EVB_API int evb_de_create(int dtype, const evb_de_config* cfg, int pop_size, int dim, evb_de* out);
EVB_API int evb_de_destroy(evb_de e);
/* de_engine::reset (de/engine.hpp:142-145): adapter to its initial state, archive emptied. */
EVB_API int evb_de_reset(evb_de e);
EVB_API int evb_de_archive_capacity(evb_de e);
EVB_API int evb_de_p_count(evb_de e);
/* de_engine::generation(pop, st, objective, lb, ub, rng) (de/engine.hpp:71-102) on a device
 * population (pop_size x ldp, row-major) and fitness vector; `objective` is evaluated with
 * problem_instance::evaluate semantics.  s may be NULL (engine-owned scratch). */
EVB_API int evb_de_generation(evb_de e, evb_problem objective, evb_scratch s, void* pop, int64_t ldp,
                              void* fitness, double lb, double ub, evb_rng rng, void* stream);
/* n consecutive generations (identical to n evb_de_generation calls): the first runs eagerly,
 * the rest replay a CUDA graph of one generation (the generation id and the word cursor are
 * device-resident), removing per-kernel launch overhead for small populations. */
EVB_API int evb_de_generations(evb_de e, evb_problem objective, evb_scratch s, void* pop, int64_t ldp,
                               void* fitness, double lb, double ub, evb_rng rng, int n, void* stream);
/* n generations on a HOST-resident population / fitness (row stride ldp elements), the shape of the
 * reference's de_engine (whose population lives on the host): one copy in, evb_de_generations on
 * the engine's own stream, one copy out; returns when the host arrays hold the result.  Fixed
 * population size only. */
EVB_API int evb_de_generations_host(evb_de e, evb_problem objective, evb_scratch s, void* pop_host, int64_t ldp,
                                    void* fitness_host, double lb, double ub, evb_rng rng, int n);
/* init_population (core/population.hpp:88-98) from the rng. */
EVB_API int evb_de_init_population(evb_de e, void* pop, int64_t ldp, double lb, double ub, evb_rng rng,
                                   void* stream);
/* de_engine::optimize (de/engine.hpp:107-133): init, evaluate, generations until max_fes. */
EVB_API int evb_de_optimize(evb_de e, evb_problem objective, evb_scratch s, void* pop, int64_t ldp,
                            void* fitness, double lb, double ub, int64_t max_fes, evb_rng rng,
                            int* best_index, double* best_fitness, int* generations, void* stream);
/* hybrid::restart_run (hybrid/restart.hpp:37-88, the "restart-lshade" preset) around this engine:
 * runs fresh engine states (adapter, archive, population size reset; the population re-drawn
 * from the continuing rng) until total_budget evaluations are spent, stopping a run once
 * stagnation_evals evaluations passed without improving the best seen by more than epsilon.
 * Recorder / parameter trace see one continuous run (generation numbers continue). */
EVB_API int evb_de_optimize_restart(evb_de e, evb_problem objective, evb_scratch s, void* pop, int64_t ldp,
                                    void* fitness, double lb, double ub, int64_t total_budget,
                                    int64_t stagnation_evals, double epsilon, evb_rng rng, double* best_fitness,
                                    int* engine_runs, int64_t* evaluations, void* stream);
/* Engine state (archive members row-major cap x dim, size; SHADE/JADE memories; write index). */
EVB_API int evb_de_get_state(evb_de e, void* archive_host, int* archive_size, void* mem_f_host,
                             void* mem_cr_host, int* write_index);
EVB_API int evb_de_set_state(evb_de e, const void* archive_host, int archive_size,
                             const void* mem_f_host, const void* mem_cr_host, int write_index);
/* Draws of the last generation: words consumed per individual, archive-victim words, the
 * Philox generation id, per-individual F, CR, donor indices (4 per individual) and jrand. */
/* evolution_state of generation-level use (core/state.hpp:10-53): budget and evaluations so far.
 * Needed before evb_de_generation when the population policy is linear_reduction (the schedule
 * reads fes / max_fes); evb_de_optimize sets it itself.  Each generation adds its trials. */
EVB_API int evb_de_set_budget(evb_de e, int64_t max_fes, int64_t fes);
/* Current population size (shrinks under linear_reduction; rows [0, size) of the caller's
 * population are the members, in the reference's order after erase_member). */
EVB_API int evb_de_pop_size(evb_de e);
/* The last generation's population size (its trial count; evb_de_last_draws reports that many
 * individuals), the size after its reduction, and the archive-shrink words consumed by
 * de_archive::set_capacity (de/strategy.hpp:40-47; Philox sub-stream 0xFFFFFFFE). */
EVB_API int evb_de_last_reduction(evb_de e, int* pop_before, int* pop_after, int64_t* shrink_words);
/* Every evaluation the engine makes (init in evb_de_optimize, trials in each generation) is
 * reported, in FE order, to recorder run `run` (run_handle::evaluate -> on_evaluate,
 * experiment/runner.hpp:38-45); r = NULL detaches. */
EVB_API int evb_de_attach_recorder(evb_de e, evb_recorder r, int run);
/* Append (generation, mu_F, mu_CR) to trace run `run` after every generation of a JADE / SHADE
 * engine (fixed adapters report nothing, as in the reference); t = NULL detaches.  The
 * generation number counts from 1 after each evb_de_optimize start (evolution_state). */
EVB_API int evb_de_attach_param_trace(evb_de e, evb_param_trace t, int run);
EVB_API int evb_de_last_draws(evb_de e, int64_t* word_counts, int64_t* archive_words, uint32_t* generation,
                              void* F_host, void* CR_host, int* idx_host, int* jrand_host);

/* K8: n_runs independent DE runs in ONE persistent launch (one CTA per run, every generation
 * inside the kernel; experiment/runner.hpp:101-160 evo_bench over a suite).  Run r evaluates
 * problems[r] (base, hybrid or composition, fp64) and draws from Philox key keys[r]; pops / fits are
 * device arrays (n_runs x pop_size x dim, n_runs x pop_size).  init != 0: draw and evaluate the
 * initial populations first (generation id gen0), then run `generations` generations (ids
 * gen0+1 ...); otherwise continue from the given populations (ids gen0 ...).  Supports the `de`
 * preset family: rand_1 / best_1, binomial, clip / midpoint_target, fixed F, CR, no archive;
 * the run state must fit in shared memory (else use evb_de_generation per run).  rec (may be
 * NULL): run r's evaluations are recorded into recorder run r, in FE order.  Asynchronous on
 * `stream` (the call returns once the launch is queued). */
EVB_API int evb_de_runs(int dtype, const evb_de_config* cfg, int n_runs, int pop_size, int dim,
                        const evb_problem* problems, const uint64_t* keys, int generations, double lb,
                        double ub, void* pops, void* fits, int init, uint32_t gen0, evb_recorder rec,
                        void* stream);

/* ---- Competitive Swarm Optimizer (pso/cso.hpp:19-99, cso_optimizer<T>) ----------------------- */

typedef struct evb_cso_s* evb_cso;

/* cso_optimizer(phi): phi finite and >= 0, pop_size even (cso.hpp:25-27, 34). */
EVB_API int evb_cso_create(int dtype, double phi, int pop_size, int dim, evb_cso* out);
EVB_API int evb_cso_destroy(evb_cso c);
/* cso_optimizer::generation (cso.hpp:31-72) — exactly the reference's generation (it is
 * data-parallel: mean of the pre-update swarm, disjoint pairs, losers read only winners).
 * X, V: pop_size x ld row-major device arrays; fitness: current fitness (losers updated). */
EVB_API int evb_cso_generation(evb_cso c, evb_problem objective, evb_scratch s, void* X, int64_t ldx, void* V,
                               int64_t ldv, void* fitness, double lb, double ub, evb_rng rng, void* stream);
/* cso_optimizer::optimize (cso.hpp:74-91): init_population, evaluate, zero velocities,
 * generations (pop_size / 2 evaluations each) while fes < max_fes; best = population::best. */
EVB_API int evb_cso_optimize(evb_cso c, evb_problem objective, evb_scratch s, void* X, int64_t ldx, void* V,
                             int64_t ldv, void* fitness, double lb, double ub, int64_t max_fes, evb_rng rng,
                             int* best_index, double* best_fitness, int* generations, void* stream);
/* Report the optimizer's evaluations (initial P in optimize, each generation's losers in pair
 * order) to recorder run `run`; r = NULL detaches. */
EVB_API int evb_cso_attach_recorder(evb_cso c, evb_recorder r, int run);

/* ---- suite-level grouped launch (experiment/runner.hpp:101-160 evo_bench) ----------------- */

/* Philox key of task t: splitmix64(master_seed ^ t), the positional analogue of
 * derive_stream(master_seed, t) (runner.hpp:119-120). */
EVB_API uint64_t evb_task_key(uint64_t master_seed, uint64_t task_index);

enum { EVB_BENCH_FORCE_ENGINE = 1 /* run every task through the per-generation engine */ };

/* evo_bench(alg = DE config `cfg` with pop_size, suite, recorder, {runs, max_fes, master_seed}):
 * problems[(p * instance_count) + i] is instance i of problem p (suite::at(p, i)); task
 * t = ((p * instance_count) + i) * runs + r runs de_engine::optimize(max_fes) from Philox key
 * evb_task_key(master_seed, t) and reports its evaluations, in FE order, to recorder run t (may
 * be NULL), then on_run_end; adaptive configurations report (generation, mu_F, mu_CR) to
 * ptrace run t (may be NULL; parameter_record).  best_host (may be NULL): each task's best.  *path_used:
 * 1 = all tasks in one persistent launch (evb_de_runs), 2 = per-task engines. */
EVB_API int evb_evo_bench_de(int dtype, const evb_de_config* cfg, int pop_size, int dim,
                             const evb_problem* problems, int problem_count, int instance_count, int runs,
                             int64_t max_fes, uint64_t master_seed, double lb, double ub, evb_recorder rec,
                             evb_param_trace ptrace, double* best_host, int flags, int* path_used,
                             void* stream);

/* Per-phase device time of each later generation (CUDA events on the launching stream, between
 * the generation's kernels): order/best, draws, trial, evaluation, selection scan, selection
 * apply.  evb_de_phase_ms synchronises and returns the last generation's phase times. */
EVB_API int evb_de_phase_timing(evb_de e, int enable);
EVB_API int evb_de_phase_ms(evb_de e, float* ms, int cap, int* n);

/* ---- PSO engine (pso/engine.hpp:33-153, pso/topology.hpp, pso/update.hpp) ------------------ */

enum evb_pso_topology { EVB_TOPO_GBEST = 0 /* "gbest" */, EVB_TOPO_LBEST_RING = 1 /* "lbest_ring" */ };
enum evb_pso_update { EVB_UPD_STANDARD = 0 /* "standard" */, EVB_UPD_SPHERICAL = 1 /* "spherical" (SPSO2011) */ };

typedef struct {
  int topology, update;
  double inertia, cognitive, social; /* swarm_params (pso/update.hpp:16-22) */
  double vmax;                       /* > 0: clamp |v| <= vmax after the velocity rule (config 3) */
  double attraction;                 /* swarm_params::attraction c of the spherical rule        */
} evb_pso_config;

typedef struct evb_pso_s* evb_pso;

EVB_API int evb_pso_create(int dtype, const evb_pso_config* cfg, int pop_size, int dim, evb_pso* out);
EVB_API int evb_pso_destroy(evb_pso s);
/* pso_engine::prepare, first call (pso/engine.hpp:40-50): personal bests <- population. */
EVB_API int evb_pso_prepare(evb_pso s, const void* X, int64_t ldx, const void* fitness, void* stream);
/* One SYNCHRONOUS generation: neighbourhood from start-of-generation pbests, velocity rule,
 * optional clamp, move + bound rule, batched evaluation, strict-< pbest update.  The stock
 * reference engine is asynchronous (pso/engine.hpp:52-82); see DESIGN.md. */
EVB_API int evb_pso_generation(evb_pso s, evb_problem objective, evb_scratch sc, void* X, int64_t ldx,
                               void* V, int64_t ldv, void* fitness, double lb, double ub, evb_rng rng,
                               void* stream);
/* A (pop_size x lda) <- U[lo, hi) from the rng (positions: init_population order; velocities). */
EVB_API int evb_pso_init_uniform(evb_pso s, void* A, int64_t lda, double lo, double hi, evb_rng rng,
                                 void* stream);
EVB_API int evb_pso_get(evb_pso s, void* pbest_host, void* pbest_fit_host, int* nb_host, uint32_t* generation);
EVB_API int evb_pso_set_pbest(evb_pso s, const void* pbest_host, const void* pbest_fit_host);
/* pso_engine::optimize (pso/engine.hpp:84-105) with the synchronous generation: init_population,
 * evaluate, zero velocities, prepare, generations while fes < max_fes; the best personal best. */
EVB_API int evb_pso_optimize(evb_pso s, evb_problem objective, evb_scratch sc, void* X, int64_t ldx, void* V,
                             int64_t ldv, void* fitness, double lb, double ub, int64_t max_fes, evb_rng rng,
                             int* best_index, double* best_fitness, int* generations, void* stream);
/* Report every evaluation (init inside optimize, each generation's particles in i order) to
 * recorder run `run`; r = NULL detaches. */
EVB_API int evb_pso_attach_recorder(evb_pso s, evb_recorder r, int run);
/* Per-phase device time (as evb_de_phase_timing): neighbourhood best, update, evaluation,
 * personal best. */
EVB_API int evb_pso_phase_timing(evb_pso s, int enable);
EVB_API int evb_pso_phase_ms(evb_pso s, float* ms, int cap, int* n);

/* evo_bench for the swarm presets (presets.hpp make_algorithm "pso" / "spso2011" / "cso"), same
 * task layout, Philox keys, recorder slots and best_host as evb_evo_bench_de; each task runs
 * evb_pso_optimize (synchronous generation) or evb_cso_optimize (the reference's
 * generation exactly, pop_size even). */
EVB_API int evb_evo_bench_pso(int dtype, const evb_pso_config* cfg, int pop_size, int dim,
                              const evb_problem* problems, int problem_count, int instance_count, int runs,
                              int64_t max_fes, uint64_t master_seed, double lb, double ub, evb_recorder rec,
                              double* best_host, void* stream);
EVB_API int evb_evo_bench_cso(int dtype, double phi, int pop_size, int dim, const evb_problem* problems,
                              int problem_count, int instance_count, int runs, int64_t max_fes,
                              uint64_t master_seed, double lb, double ub, evb_recorder rec, double* best_host,
                              void* stream);

/* Kernel launches this library has issued on the calling thread (monotonic counter; used by
 * bench.py to report gpu_launches inside its timed region). */
EVB_API int evb_launch_count(void);

/* Live roofline denominator: which = 0 -> FP64 tensor (DMMA m8n8k4) TFLOP/s, which = 1 -> FP32
 * FFMA TFLOP/s, measured by a throughput kernel over every SM (best of 3 launches). */
EVB_API int evb_probe_peak_tflops(int which, int iters, double* tflops);

#ifdef __cplusplus
} /* extern "C" */
#endif

#endif /* EVB_H_ */

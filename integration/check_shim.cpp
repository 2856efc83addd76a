// Compile check of the reference-side shim against the reference's own headers
// (tests/test_integration_shim.py): instantiates every entry point.
#include "dc_engine_b200.hpp"

void shim_entry_points(const topopt::GridModel& g, const topopt::ActionSet& a, const topopt::QdConfig& q) {
  topopt::b200::GpuDcContext ctx(g, a, topopt::DcConfig{});
  std::vector<topopt::Genome> gs{topopt::Genome::empty(q.n_a, q.n_d)};
  std::vector<topopt::ScoreVector> s = ctx.evaluate_batch(gs, q.batch_size);
  topopt::ScoreVector one = ctx.evaluate(gs[0]);
  std::atomic<bool> stop{false};
  topopt::OptimizerStats st = topopt::b200::run_optimizer_gpu(ctx, q, [](topopt::RepertoireSnapshot) {}, &stop);
  (void)s;
  (void)one;
  (void)st;
}

void shim_ac_entry_points(const topopt::GridModel& g, const topopt::ActionSet& a, const topopt::DcContext& dc,
                          const topopt::b200::GpuDcContext& gdc) {
  topopt::b200::GpuAcValidator val(g, a, dc, topopt::AcConfig{}, &gdc);
  std::vector<topopt::Candidate> cs{topopt::Candidate{topopt::Genome::empty(3, 2), topopt::ScoreVector{}}};
  topopt::EliminationOutcome out = val.eliminate(cs);
  std::vector<topopt::RejectionReason> wk = val.worst_k_check(cs);
  std::vector<topopt::ValidationRecord> full = val.full_validation(cs);
  std::vector<topopt::ValidationRecord> recs = val.validate_queue(cs);
  topopt::ValidationRecord one = val.validate(cs[0]);
  val.record_elimination(cs[0], topopt::RejectionReason::EliminatedSimilar);
  (void)out;
  (void)wk;
  (void)full;
  (void)recs;
  (void)one;
  (void)val.baseline_lambda_o();
  (void)val.records();
}

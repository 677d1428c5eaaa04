// costs.cc — O (memory), c (layer time) and R (relayout) of Eq. 1.
//
// These must be bit-identical to the reference cost model (proj/src/cost_model.cc:92-241),
// because every DP tie-break downstream compares these doubles.  The expressions below keep
// the reference's operation order and operand types exactly; the build disables FMA
// contraction (-ffp-contract=off) for the same reason.
#include <algorithm>
#include <cmath>

#include "parplan/cost_model.h"

namespace parplan {

int MemoryUnits(double bytes, int64_t granularity_bytes) {
  return static_cast<int>(std::ceil(bytes / static_cast<double>(granularity_bytes)));
}

double CollectiveVolumeBytes(CollectiveKind kind, int degree, double payload_bytes) {
  if (degree < 1) throw ValidationError("collective: degree must be >= 1");
  if (!(payload_bytes >= 0.0)) throw ValidationError("collective: payload must be >= 0");
  if (degree == 1) return 0.0;
  // (payload * (d-1)) / d, evaluated left to right
  const double moved = payload_bytes * static_cast<double>(degree - 1) / static_cast<double>(degree);
  return kind == CollectiveKind::kAllReduce ? 2.0 * moved : moved;
}

namespace {

struct Split {
  int dp, sdp, tp;
  int data;                   // dp * sdp: how many ways the batch is split
  double samples_per_device;  // batch / data
};

// nullopt when there are more data replicas than samples.
std::optional<Split> SplitOf(const HybridStrategy& s, int batch) {
  const HybridStrategy::Degrees d = s.DimDegrees();
  Split sp{d.dp, d.sdp, d.tp, d.dp * d.sdp, 0.0};
  if (sp.data > batch) return std::nullopt;
  sp.samples_per_device = static_cast<double>(batch) / static_cast<double>(sp.data);
  return sp;
}

}  // namespace

std::optional<MemoryBreakdown> EstimateMemory(const LayerSpec& layer,
                                              const HybridStrategy& strategy,
                                              int batch_per_group, const CostProfile& profile) {
  if (batch_per_group < 1) throw ValidationError("memory: batch_per_group must be >= 1");
  const auto sp = SplitOf(strategy, batch_per_group);
  if (!sp) return std::nullopt;
  const double rho = profile.tp_activation_replication;
  MemoryBreakdown m;
  m.params_bytes = static_cast<double>(layer.param_bytes) / static_cast<double>(sp->tp * sp->sdp);
  m.grads_bytes = m.params_bytes;
  m.optimizer_bytes = m.params_bytes * profile.optimizer_state_multiplier;
  const double act_factor = (1.0 - rho) / static_cast<double>(sp->tp) + rho;
  m.activation_bytes =
      static_cast<double>(layer.activation_bytes_per_sample) * sp->samples_per_device * act_factor;
  return m;
}

std::optional<LayerCost> EstimateLayerCost(const LayerSpec& layer, const HybridStrategy& strategy,
                                           int batch_per_group, double bandwidth_gbps,
                                           const CostProfile& profile) {
  if (batch_per_group < 1) throw ValidationError("cost: batch_per_group must be >= 1");
  if (!(bandwidth_gbps > 0.0)) throw ValidationError("cost: bandwidth must be > 0");
  const auto sp = SplitOf(strategy, batch_per_group);
  if (!sp) return std::nullopt;
  const double act = static_cast<double>(layer.activation_bytes_per_sample);
  const double params = static_cast<double>(layer.param_bytes);

  LayerCost c;
  c.forward_ms = layer.fwd_time_per_sample_ms * sp->samples_per_device;
  c.backward_ms = c.forward_ms * profile.backward_multiplier;

  // serial: TP activation all-reduce (once in fwd, once in bwd), SDP param gather before fwd
  const double tp_ms = BytesToMs(
      CollectiveVolumeBytes(CollectiveKind::kAllReduce, sp->tp,
                            act * sp->samples_per_device * profile.tp_activation_replication),
      bandwidth_gbps);
  const double tp_shard = params / static_cast<double>(sp->tp);
  const double gather_ms =
      BytesToMs(CollectiveVolumeBytes(CollectiveKind::kAllGather, sp->sdp, tp_shard),
                bandwidth_gbps);

  // overlappable with backward: DP all-reduce of the owned shard, SDP re-gather + scatter
  const double owned = params / static_cast<double>(sp->tp * sp->sdp);
  const double grad_ms =
      BytesToMs(CollectiveVolumeBytes(CollectiveKind::kAllReduce, sp->dp, owned), bandwidth_gbps) +
      gather_ms +
      BytesToMs(CollectiveVolumeBytes(CollectiveKind::kReduceScatter, sp->sdp, tp_shard),
                bandwidth_gbps);

  const bool both = c.backward_ms > 0.0 && grad_ms > 0.0;
  const double bwd_segment =
      both ? std::max(c.backward_ms, grad_ms) * profile.overlap_slowdown : c.backward_ms + grad_ms;

  c.comm_ms_unoverlapped = tp_ms + tp_ms + gather_ms + grad_ms;
  c.total_ms = c.forward_ms + gather_ms + tp_ms + tp_ms + bwd_segment;
  return c;
}

double TransformationCostMs(const LayerSpec& layer, const HybridStrategy& prev,
                            const HybridStrategy& cur, int batch_per_group,
                            double bandwidth_gbps) {
  if (prev.group_size != cur.group_size)
    throw ValidationError("transformation: neighboring strategies must share group size");
  if (prev == cur) return 0.0;
  const HybridStrategy::Degrees a = prev.DimDegrees();
  const HybridStrategy::Degrees b = cur.DimDegrees();
  if (a.dp == b.dp && a.sdp == b.sdp && a.tp == b.tp) return 0.0;  // reorder only
  const double act_delta = std::abs(1.0 / static_cast<double>(b.dp * b.sdp) -
                                    1.0 / static_cast<double>(a.dp * a.sdp));
  const double act_bytes = static_cast<double>(layer.activation_bytes_per_sample) *
                           static_cast<double>(batch_per_group) * act_delta;
  const double widen = std::max(0.0, 1.0 / static_cast<double>(b.tp * b.sdp) -
                                         1.0 / static_cast<double>(a.tp * a.sdp));
  const double param_bytes = static_cast<double>(layer.param_bytes) * widen;
  return BytesToMs(act_bytes + param_bytes, bandwidth_gbps);
}

}  // namespace parplan

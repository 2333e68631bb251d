// The reference-side shim of INTEGRATION.md §2-§4, as compiled code: the B200 library behind the
// reference's own objective plugin (proj/include/adpsgd/objectives.hpp:45-69) and error types
// (proj/include/adpsgd/errors.hpp:9-46). Built by tools/shim/Makefile against the reference's
// headers where they lie (plus the storage-only Eigen stand-in) -- this is what a reference
// maintainer would add to proj/, not part of this repository's product path.
#pragma once
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "adpsgd/errors.hpp"
#include "adpsgd/objectives.hpp"
#include "adpsgd_b200.h"

namespace b200 {

// adpsgd_status -> the reference's exception taxonomy (errors.hpp:9-46)
inline void check(int rc) {
    if (rc == ADPSGD_OK) return;
    const std::string m = adpsgd_last_error();
    switch (rc) {
        case ADPSGD_E_INVALID_ORDER: throw adpsgd::InvalidOrderError(m);
        case ADPSGD_E_DIMENSION: throw adpsgd::DimensionError(m);
        case ADPSGD_E_OUT_OF_REGIME: throw adpsgd::OutOfRegimeError(m);
        case ADPSGD_E_NUMERICAL: throw adpsgd::NumericalError(m);
        case ADPSGD_E_SYNC_VIOLATION: throw adpsgd::SyncViolationError(m);
        case ADPSGD_E_STALENESS_OVERFLOW: throw adpsgd::StalenessOverflowError(m);
        case ADPSGD_E_INVALID_STATE: throw adpsgd::InvalidStateError(m);
        case ADPSGD_E_CONFIG: throw adpsgd::ConfigError(m);
        default: throw std::runtime_error("CUDA/NCCL: " + m);
    }
}

// Objective::gradient / loss / heldout_loss of the BLSTM on the device (adpsgd_gradient,
// adpsgd_eval_loss); the dataset is the device-resident copy of feats / labels.
class LstmObjective : public adpsgd::objectives::Objective {
  public:
    LstmObjective(const adpsgd_model_desc& m, int32_t precision, int batch, const std::vector<float>& feats,
                  const std::vector<int32_t>& labels, int n_seg, int train_count)
        : n_seg_(n_seg), train_count_(train_count) {
        adpsgd_config c{};
        c.model = m;
        c.precision = precision;
        c.strategy = ADPSGD_SDPSGD;
        c.learners = 1;
        c.local_learners = 1;
        c.batch = batch;
        check(adpsgd_ctx_create(&c, &ctx_));
        check(adpsgd_set_dataset(ctx_, feats.data(), labels.data(), n_seg, train_count));
        dimension_ = static_cast<int>(adpsgd_param_count(&m));
    }
    ~LstmObjective() override { adpsgd_ctx_destroy(ctx_); }
    LstmObjective(const LstmObjective&) = delete;
    LstmObjective& operator=(const LstmObjective&) = delete;

    adpsgd::objectives::Vec gradient(const adpsgd::objectives::Vec& w,
                                     const adpsgd::objectives::SampleBatch& b) const override {
        adpsgd::objectives::Vec g(dimension_);
        double loss = 0.0;
        check(adpsgd_gradient(ctx_, w.data(), b.indices.data(), b.size(), g.data(), &loss));
        return g;
    }
    double loss(const adpsgd::objectives::Vec& w, const adpsgd::objectives::SampleBatch& b) const override {
        double loss = 0.0;
        check(adpsgd_eval_loss(ctx_, w.data(), b.indices.data(), b.size(), &loss));
        return loss;
    }
    double heldout_loss(const adpsgd::objectives::Vec& w) const override {
        std::vector<int> idx;
        for (int i = train_count_; i < n_seg_; ++i) idx.push_back(i);
        double loss = 0.0;
        check(adpsgd_eval_loss(ctx_, w.data(), idx.data(), static_cast<int32_t>(idx.size()), &loss));
        return loss;
    }

  private:
    adpsgd_ctx* ctx_ = nullptr;
    int n_seg_, train_count_;
};

}  // namespace b200

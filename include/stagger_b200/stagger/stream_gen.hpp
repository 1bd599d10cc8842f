// Drop-in subset of stagger/stream_gen.hpp: the pull-based FrameSource /
// FrameSink types and vector_source (stream_gen.hpp:15-62).
#pragma once

#include <functional>
#include <memory>
#include <optional>
#include <vector>

#include "stagger/core.hpp"

namespace stagger {

using FrameSource = std::function<std::optional<Frame>()>;
using FrameSink = std::function<void(const Frame&)>;

inline FrameSource vector_source(std::vector<Frame> frames) {
    auto data = std::make_shared<std::vector<Frame>>(std::move(frames));
    auto idx = std::make_shared<std::size_t>(0);
    return [data, idx]() -> std::optional<Frame> {
        if (*idx >= data->size()) return std::nullopt;
        return (*data)[(*idx)++];
    };
}

}  // namespace stagger

// fodg drop-in (B200 engine): the few controls the device engine adds to the
// reference's API.  Nothing here is needed by code written against the
// reference; it exists for callers that want to manage the device state.
#pragma once

#include <cstddef>
#include <cstdint>

namespace fodg::b200 {

/// batch_search / search_one keep the uploaded (Graph, Dataset) pair on the
/// device between calls.  Default rule: an entry is reused only when the
/// buffers' addresses, shapes AND full-content hashes match the upload, so an
/// in-place edit of graph.ids or a new Dataset at a recycled address is always
/// re-uploaded.  With CAGRA_INDEX_CACHE=identity the hash is skipped (address
/// and shape only); a caller that then mutates a searched Graph in place must
/// call this to drop every cached device index.
void invalidate_index_cache();

/// The content hash used by the cache (exposed for tests).
std::uint64_t host_content_hash(const void* p, std::size_t bytes);

}  // namespace fodg::b200

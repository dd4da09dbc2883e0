"""TEST INFRASTRUCTURE ONLY (parity checker, CPU baseline).  Never imported by the product."""
